// Band-kernel instantiations: padded label stride Ms = 256, max domain.
#include "fused_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band_dom<256, SBP_MAX>(int, int, int);
template FusedLaunchFn pick_fused<256, SBP_MAX>(int, bool);
}
