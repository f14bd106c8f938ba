// Band-kernel instantiations for one padded label stride SBP_MS and domain
// SBP_DOM, split into parts so the build compiles them in parallel
// (the Makefile compiles this file once per (Ms, domain, part)):
//   part 0: register-loaded unrolled VL=8 kernels + the variant dispatcher
//   part 4: register-loaded unrolled VL=16 kernels
//   part 1: rolled kernels (one band copy for the four directions)
//   part 2 / 5: TMA-staged VL=8 / VL=16 kernels
//   part 3: temporally blocked (fused) kernels
#include "fused_kernel.cuh"

#if !defined(SBP_MS) || !defined(SBP_DOM) || !defined(SBP_PART)
#error "compile with -DSBP_MS=<Ms> -DSBP_DOM=<SBP_SUM|SBP_MAX> -DSBP_PART=<0..5>"
#endif

namespace sbp {

#if SBP_PART == 0
extern template BandLaunchFn pick_band_r<SBP_MS, SBP_DOM, 16, false>(int);
extern template BandLaunchFn pick_band_r<SBP_MS, SBP_DOM, 8, true>(int);
extern template BandLaunchFn pick_band_r<SBP_MS, SBP_DOM, 16, true>(int);
extern template BandLaunchFn pick_band_staged_r<SBP_MS, SBP_DOM, 8, 2>(int);
extern template BandLaunchFn pick_band_staged_r<SBP_MS, SBP_DOM, 16, 1>(int);
template BandLaunchFn pick_band_r<SBP_MS, SBP_DOM, 8, false>(int);
template BandLaunchFn pick_band_dom<SBP_MS, SBP_DOM>(int, int, int);
#elif SBP_PART == 1
template BandLaunchFn pick_band_r<SBP_MS, SBP_DOM, 8, true>(int);
template BandLaunchFn pick_band_r<SBP_MS, SBP_DOM, 16, true>(int);
#elif SBP_PART == 2
template BandLaunchFn pick_band_staged_r<SBP_MS, SBP_DOM, 8, 2>(int);
#elif SBP_PART == 3
template FusedLaunchFn pick_fused<SBP_MS, SBP_DOM>(int, bool);
#elif SBP_PART == 4
template BandLaunchFn pick_band_r<SBP_MS, SBP_DOM, 16, false>(int);
#elif SBP_PART == 5
template BandLaunchFn pick_band_staged_r<SBP_MS, SBP_DOM, 16, 1>(int);
#endif

}  // namespace sbp
