// Sequential-sweep (chain) kernel instantiations: Ms = 8, max domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<8, SBP_MAX>(int, int);
}
