// Band-kernel instantiations: padded label stride Ms = 16, sum domain.
#include "fused_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band_dom<16, SBP_SUM>(int, int, int);
template FusedLaunchFn pick_fused<16, SBP_SUM>(int, bool);
}
