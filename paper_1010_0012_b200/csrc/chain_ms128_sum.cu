// Sequential-sweep (chain) kernel instantiations: Ms = 128, sum domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<128, SBP_SUM>(int, int);
}
