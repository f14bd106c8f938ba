// Band-kernel instantiations: padded label stride Ms = 16, max domain.
#include "fused_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band_dom<16, SBP_MAX>(int, int, int);
template FusedLaunchFn pick_fused<16, SBP_MAX>(int, bool);
}
