// Sequential-sweep (chain) kernel instantiations: Ms = 32, max domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<32, SBP_MAX>(int, int);
}
