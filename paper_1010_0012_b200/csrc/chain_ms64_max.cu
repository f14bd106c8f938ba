// Sequential-sweep (chain) kernel instantiations: Ms = 64, max domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<64, SBP_MAX>(int, int);
}
