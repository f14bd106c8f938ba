// Band-kernel instantiations for padded label stride Ms = 16.
#include "band_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band<16>(int, int, int);
}
