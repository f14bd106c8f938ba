// Sequential-sweep (chain) kernel instantiations: Ms = 256, sum domain.
#include "chain_kernel.cuh"
namespace sbp {
template BandLaunchFn pick_chain<256, SBP_SUM>(int, int);
}
