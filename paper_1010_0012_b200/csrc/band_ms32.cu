// Band-kernel instantiations for padded label stride Ms = 32.
#include "band_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_band<32>(int, int, int);
}
