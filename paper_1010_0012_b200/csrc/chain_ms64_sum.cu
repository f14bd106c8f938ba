// Sequential-sweep (chain) kernel instantiations: Ms = 64, sum domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<64, SBP_SUM>(int, int);
}
