// Shared-memory-tap band kernel instantiations for one padded label stride
// SBP_MS and domain SBP_DOM (the Makefile compiles this file once per pair).
#include "tap_kernel.cuh"

#if !defined(SBP_MS) || !defined(SBP_DOM)
#error "compile with -DSBP_MS=<Ms> -DSBP_DOM=<SBP_SUM|SBP_MAX>"
#endif

namespace sbp {
template BandLaunchFn pick_band_tap<SBP_MS, SBP_DOM>(int, int, int, int);
}
