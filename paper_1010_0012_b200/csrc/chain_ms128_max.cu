// Sequential-sweep (chain) kernel instantiations: Ms = 128, max domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<128, SBP_MAX>(int, int);
}
