// Sequential-sweep (chain) kernel instantiations: Ms = 8, sum domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<8, SBP_SUM>(int, int);
}
