// Sequential-sweep (chain) kernel instantiations: Ms = 16, max domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<16, SBP_MAX>(int, int);
}
