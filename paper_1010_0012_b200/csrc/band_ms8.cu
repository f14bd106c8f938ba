// Band-kernel instantiations for padded label stride Ms = 8.
#include "band_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band<8>(int, int, int);
}
