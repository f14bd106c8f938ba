// Band-kernel instantiations for padded label stride Ms = 128.
#include "band_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band<128>(int, int, int);
}
