// Band-kernel instantiations: padded label stride Ms = 64, max domain.
#include "fused_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band_dom<64, SBP_MAX>(int, int, int);
template FusedLaunchFn pick_fused<64, SBP_MAX>(int, bool);
}
