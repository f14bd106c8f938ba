// Band-kernel instantiations: padded label stride Ms = 128, max domain.
#include "fused_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band_dom<128, SBP_MAX>(int, int, int);
template FusedLaunchFn pick_fused<128, SBP_MAX>(int, bool);
}
