// Sequential-sweep (chain) kernel instantiations: Ms = 16, sum domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<16, SBP_SUM>(int, int);
}
