// Temporally blocked synchronous iterations (sm_100a): T consecutive
// synchronous iterations in ONE persistent launch, as a wavefront over rows,
// so the messages of the intermediate iterations live in L2 instead of HBM.
//
// Level l of a launch is iteration (iteration0 + l); it reads buffer l % 2
// and writes buffer (l + 1) % 2 (relative to the launch's input buffer).
// Work units are (level l, local row r, column segment s) ordered by
// tau = r + l * D (then level, then segment); level l at row r needs level
// l-1 finished at rows r-1..r+1 (columns s-1..s+1 of row r, column s of rows
// r +- 1): those units have tau' <= tau + 1 - D < tau for D >= 2, i.e. they
// come earlier in the order.  The same waits also cover every write-after-
// read hazard of the ping-pong buffers: level l+1 writes into rows q-1..q+1
// of buffer in(l) only after level l finished reading them.  Warp w runs
// units w, w + G, ... in order; the launch is cooperative (all warps
// co-resident), so the smallest unfinished unit always has its inputs and
// its warp at it: no deadlock.
//
// A unit is one warp's worth of pixels (rounds x 32/LP); completion is an
// epoch stamp per unit (release store by lane 0 after a warp barrier;
// acquire loads by the waiting warp), so the stamp array is never cleared.  Units of level >= 1 read their messages with
// L1-bypassing loads (ld.global.cg: the data was written in this launch) and
// afterwards discard those L2 lines (discard.global.L2): the intermediate
// messages are dead once read, so they are never written back to HBM.  Per
// launch HBM moves the input messages and the unaries once and the output
// messages once, whatever T: B = 4 M (N + 2E) bytes per T iterations.
//
// The per-node arithmetic is band_group_body() of the one-iteration kernel,
// so results are bit-identical to T separate launches.
#pragma once

#include "band_kernel.cuh"

namespace sbp {

constexpr int SBP_FUSE_MAX = 4;   // levels per launch

struct FusedArgs {
    IterCtx lev[SBP_FUSE_MAX];   // per level: in / out buffer, iteration, first
    unsigned *stamps;            // [SBP_FUSE_MAX][rows][nseg] epoch stamps
    unsigned epoch;
    int T, D, nseg, seg_px, rounds;
    long long units;
};

template <int N>
struct Vec8LoaderCG {
    static __device__ __forceinline__ void load(float (&dst)[N], const float *src) {
#pragma unroll
        for (int c = 0; c < N / 8; ++c) {
            const float *p = src + 8 * c;
            asm volatile(
                "ld.global.cg.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=f"(dst[8 * c + 0]), "=f"(dst[8 * c + 1]), "=f"(dst[8 * c + 2]),
                  "=f"(dst[8 * c + 3]), "=f"(dst[8 * c + 4]), "=f"(dst[8 * c + 5]),
                  "=f"(dst[8 * c + 6]), "=f"(dst[8 * c + 7])
                : "l"(p)
                : "memory");
        }
    }
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void discard_l2(const void *p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

template <int DOM, int VL, int LP, int R, bool ROLLED>
__global__ void __launch_bounds__(128, (VL == 8 ? (DOM == SBP_SUM && R <= 7 ? 6 : 4) : (R <= 8 ? 4 : 3)))
band_fused_kernel(const __grid_constant__ BandArgs a, const __grid_constant__ FusedArgs f) {
    constexpr int PPW = 32 / LP;   // pixels per warp and round
    const int lane = threadIdx.x & 31;
    const int j = lane % LP;
    const int x0 = j * VL;
    const int rows = a.lr_end - a.lr_begin;
    const long long W = a.W;
    // one warp = one work unit: no CTA barriers (they were the top stall).
    // Unit u = q * nseg + seg with q = tau * T + l, walked incrementally
    // (u += nwarps) so the loop carries no 64-bit divisions.
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    const int u0 = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int dq = nwarps / f.nseg, dseg = nwarps % f.nseg;
    int q = u0 / f.nseg, seg = u0 % f.nseg;
    for (int u = u0; u < (int)f.units; u += nwarps, seg += dseg, q += dq) {
        if (seg >= f.nseg) { seg -= f.nseg; ++q; }
        const int tau = q / f.T;
        const int l = q - tau * f.T;
        const int rr = tau - l * f.D;                    // 0-based local row
        if (rr < 0 || rr >= rows) continue;              // warp-uniform
        const IterCtx it = f.lev[l];
        if (l > 0) {
            // lanes 0..4 wait for the five producer units of level l-1
            if (lane < 5) {
                int pr = rr;
                int ps = seg;
                if (lane == 0) pr = rr - 1;
                else if (lane == 1) pr = rr + 1;
                else ps = seg + (lane - 3);   // lanes 2, 3, 4: seg-1, seg, seg+1
                if (pr >= 0 && pr < rows && ps >= 0 && ps < f.nseg) {
                    const unsigned *st =
                        f.stamps + ((long long)(l - 1) * rows + pr) * f.nseg + ps;
                    while (ld_acquire(st) != f.epoch) __nanosleep(20);
                }
            }
            __syncwarp();
        }
        const int lr = a.lr_begin + (int)rr;
        const long long r = (long long)a.r0 + lr - 1;
        for (int k = 0; k < f.rounds; ++k) {
            long long c = (long long)seg * f.seg_px + (long long)k * PPW + lane / LP;
            const bool valid = c < W;
            if (!valid) c = W - 1;
            const long long node_l = (long long)lr * W + c;
            float g[VL], m0[VL], m1[VL], m2[VL], m3[VL];
            Vec8Loader<VL>::load(g, a.values + ((long long)(lr - 1) * W + c) * a.Ms + x0);
            const float *mi = it.msgs_in + node_l * a.Ms + x0;
            if (it.first) {
                const bool ghost[4] = {r == 0, c == 0, c == W - 1, r == a.H - 1};
                float *mm[4] = {m0, m1, m2, m3};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float real = DOM == SBP_SUM ? (ghost[q] ? 1.0f : 1.0f / (float)a.M) : 0.0f;
#pragma unroll
                    for (int i = 0; i < VL; ++i)
                        mm[q][i] = x0 + i < a.M ? real : (DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf());
                }
            } else {
                // level 0 reads the previous launch's messages, but level 2
                // rewrites that buffer within this launch: no .nc (read-only
                // for the kernel's lifetime) loads for messages at any level
                Vec8LoaderCG<VL>::load(m0, mi);
                Vec8LoaderCG<VL>::load(m1, mi + a.slot_stride);
                Vec8LoaderCG<VL>::load(m2, mi + 2 * a.slot_stride);
                Vec8LoaderCG<VL>::load(m3, mi + 3 * a.slot_stride);
            }
            if constexpr (ROLLED)
                band_group_body_rolled<DOM, VL, LP, R>(a, it, g, m0, m1, m2, m3, j, x0, valid, node_l, r, c);
            else
                band_group_body<DOM, VL, LP, R>(a, it, g, m0, m1, m2, m3, j, x0, valid, node_l, r, c);
            if (l > 0 && valid && ((x0 * 4) & 127) == 0) {
                // the level's inputs are dead now (the next writer is level
                // l+1): drop them from L2 without a write-back.  Ghost slots
                // (no neighbour) are constants and stay.
                if (r > 0) discard_l2(mi);
                if (c > 0) discard_l2(mi + a.slot_stride);
                if (c < W - 1) discard_l2(mi + 2 * a.slot_stride);
                if (r < a.H - 1) discard_l2(mi + 3 * a.slot_stride);
            }
        }
        // release: cumulative over the warp's stores (bar.warp.sync orders
        // them before lane 0's release store)
        __syncwarp();
        if (lane == 0) st_release(f.stamps + ((long long)l * rows + rr) * f.nseg + seg, f.epoch);
    }
}

using FusedLaunchFn = cudaError_t (*)(const BandArgs &, FusedArgs &, cudaStream_t);

template <int DOM, int VL, int LP, int R, bool ROLLED>
cudaError_t launch_band_fused(const BandArgs &a, FusedArgs &f, cudaStream_t s) {
    constexpr int PPW = 32 / LP;
    static int resident = 0, sms = 0;
    if (!resident) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, band_fused_kernel<DOM, VL, LP, R, ROLLED>,
                                                      128, 0);
        if (resident < 1) resident = 1;
    }
    f.seg_px = PPW * f.rounds;
    f.nseg = (int)((a.W + f.seg_px - 1) / f.seg_px);
    const long long rows = a.lr_end - a.lr_begin;
    f.units = (rows + (long long)(f.T - 1) * f.D) * f.T * f.nseg;
    if (f.units >= (1LL << 31) - (1LL << 24)) return cudaErrorInvalidValue;   // 32-bit unit walk
    long long blocks = (long long)sms * resident;
    if (blocks > f.units) blocks = f.units;
    if (blocks <= 0) return cudaSuccess;
    void *args[] = {(void *)&a, (void *)&f};
    return cudaLaunchCooperativeKernel((const void *)band_fused_kernel<DOM, VL, LP, R, ROLLED>,
                                       dim3((unsigned)blocks), dim3(128), args, 0, s);
}

// Fused kernels exist for the register-loaded variants at R in {1..4, 7, 8}
// (the BASELINE bands up to m = 17; wider bands measured slower fused), with the
// lane width the one-iteration kernel uses (VL = 16 for sum, Ms >= 128,
// R <= 8; else 8); `rolled` (symmetric potentials) for R in {4, 7, 8}.
// Ms >= 32 only: a node's slot vector must cover whole 128-byte L2 lines for
// the discards (smaller label sets run the one-iteration kernel).
template <int MS, int DOM>
FusedLaunchFn pick_fused(int R, bool rolled) {
    if constexpr (MS < 32) {
        return nullptr;
    } else {
        switch (R) {
#define SBP_CASE(RR)                                                                  \
    case RR:                                                                          \
        if constexpr (RR < MS && (RR <= 4 || RR == 7 || RR == 8)) {                   \
            constexpr int VLF = (DOM == SBP_SUM && MS >= 128 && RR <= 8) ? 16 : 8;    \
            if constexpr (RR == 4 || RR == 7 || RR == 8)                              \
                if (rolled) return &launch_band_fused<DOM, VLF, MS / VLF, RR, true>;  \
            return &launch_band_fused<DOM, VLF, MS / VLF, RR, false>;                 \
        }                                                                             \
        return nullptr;
            SBP_BAND_RADII(SBP_CASE)
#undef SBP_CASE
        default: return nullptr;
        }
    }
}

}  // namespace sbp
