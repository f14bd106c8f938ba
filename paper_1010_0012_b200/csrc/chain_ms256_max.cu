// Sequential-sweep (chain) kernel instantiations: Ms = 256, max domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<256, SBP_MAX>(int, int);
}
