// Sequential-sweep (chain) kernel instantiations: Ms = 32, sum domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<32, SBP_SUM>(int, int);
}
