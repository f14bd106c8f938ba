// Band-kernel instantiations: padded label stride Ms = 64, max domain.
#include "band_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band_dom<64, SBP_MAX>(int, int, int);
}
