// Band-kernel instantiations for padded label stride Ms = 64.
#include "band_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band<64>(int, int, int);
}
