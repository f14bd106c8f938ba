// Band-kernel instantiations for padded label stride Ms = 256.
#include "band_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band<256>(int, int, int);
}
