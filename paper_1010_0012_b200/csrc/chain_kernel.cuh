// Canonical sequential sweep on the GPU: the reference's in-place
// directional passes (numba_kernels.py:274-407 `grid_pass_*`, bp.py:492-503
// `_run_grid`).
//
// A pass (L->R, R->L, T->B, B->T) is a set of independent chains -- the rows
// (horizontal passes) or columns (vertical passes) -- each a sequence of
// dependent message updates: the message from node src to src+step becomes
// the incoming slot `wslot` of src+step, which the next step of the same chain
// reads.  Chains only read slots no other chain of the pass writes, so they
// run in parallel: LP lanes per chain, the chained message carried in
// registers, the next CHAIN_LA nodes' unary and two other incoming vectors
// in a register ring (loaded CHAIN_LA steps ahead), L2-prefetched CHAIN_PF
// steps ahead.  The per-message
// arithmetic is band_message() of the synchronous kernel: same products in
// the reference order, same error-free max-sum h, same normalisation.
#pragma once

#include "band_kernel.cuh"

namespace sbp {

// register lookahead (steps): 3 for sum-product (C4 5.11 vs 6.33 ms per
// sweep, C5 T=9 2.93 vs 3.65; profiles/r01_ab_seq.txt); max-sum keeps one
// step (its TwoSum state leaves no registers: 3 steps measured 4 % slower)
template <int DOM, int VL>
constexpr int chain_lookahead() { return DOM == SBP_SUM ? (VL == 8 ? 3 : 1) : 1; }
constexpr int CHAIN_PF = 12;   // L2 prefetch distance (steps)

// Geometry of pass `dir` (numba_kernels.py:230-245 `_grid_step`).
struct PassGeom {
    long long n_lines, line_len, line_stride, step, origin;
    int excl, wslot;
};

__device__ __forceinline__ PassGeom pass_geom(int dir, long long H, long long W) {
    PassGeom g;
    if (dir == 0) { g.n_lines = H; g.line_len = W - 1; g.line_stride = W; g.step = 1; g.origin = 0; g.excl = 2; g.wslot = 1; }
    else if (dir == 1) { g.n_lines = H; g.line_len = W - 1; g.line_stride = W; g.step = -1; g.origin = W - 1; g.excl = 1; g.wslot = 2; }
    else if (dir == 2) { g.n_lines = W; g.line_len = H - 1; g.line_stride = 1; g.step = W; g.origin = 0; g.excl = 3; g.wslot = 0; }
    else { g.n_lines = W; g.line_len = H - 1; g.line_stride = 1; g.step = -W; g.origin = (H - 1) * W; g.excl = 0; g.wslot = 3; }
    return g;
}

// h in the reference order: unary, then slots 0..3 ascending, skipping excl
// (numba_kernels.py:194-227).  Max-sum: the same error-free TwoSum chain as
// the synchronous kernel (an identical sequence of roundings), then the shift.
template <int DOM, int VL, int LP>
__device__ __forceinline__ void chain_h(const float (&g)[VL], const float (&ma)[VL],
                                        const float (&mb)[VL], const float (&mc)[VL], int dir,
                                        float (&h)[VL]) {
    // the three included slots in ascending order are (ma, mb, mc); see
    // chain_pass_kernel for the assignment per pass
    if (DOM == SBP_SUM) {
        vmul(h, g, ma);
        vmul(h, h, mb);
        vmul(h, h, mc);
    } else {
        float s[VL], e[VL];
        vtwo_sum(g, ma, s, e);
        vtwo_sum_acc(s, mb, e, e);
        vtwo_sum_acc(s, mc, e, e);
        shift_compensated<VL, LP>(s, e, h);
    }
}

template <int DOM, int VL, int LP, int R>
__global__ void __launch_bounds__(128) chain_pass_kernel(const __grid_constant__ BandArgs a) {
    constexpr int CPW = 32 / LP;   // chains per warp
    constexpr int CHAIN_LA = chain_lookahead<DOM, VL>();
    const int dir = a.pass;
    const PassGeom geo = pass_geom(dir, a.H, a.W);
    const int lane = threadIdx.x & 31;
    const int j = lane % LP;
    const int x0 = j * VL;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (warp * CPW >= geo.n_lines) return;   // warp-uniform
    long long line = warp * CPW + lane / LP;
    const bool valid = line < geo.n_lines;
    if (!valid) line = geo.n_lines - 1;
    const long long src0 = line * geo.line_stride + geo.origin;
    const long long W = a.W;
    float *msgs = a.msgs_out;   // in place, [4][H+2][W][Ms]; node n lives at local n + W
    const long long S = a.slot_stride;
    // slots read from memory besides the chained one (fixed per pass direction)
    const int sa = (dir <= 1) ? 0 : 1;
    const int sb = (dir <= 1) ? 3 : 2;
    auto node_ptr = [&](int slot, long long n) { return msgs + slot * S + (n + W) * a.Ms + x0; };

    // the chained message lives in registers; the next CHAIN_LA nodes' unary
    // and two other incoming vectors (independent of the chain) sit in a
    // register ring, loaded CHAIN_LA steps ahead; L2 prefetch CHAIN_PF ahead
    float chain[VL], gq[CHAIN_LA][VL], aq[CHAIN_LA][VL], bq[CHAIN_LA][VL];
    float dmax = 0.0f;   // convergence test (BandArgs::delta): |new - old| in place
    Vec8Loader<VL>::load(chain, node_ptr(geo.wslot, src0));
    const long long len = geo.line_len;
#pragma unroll
    for (int k = 0; k < CHAIN_LA; ++k) {
        if (k < len) {
            const long long n = src0 + k * geo.step;
            Vec8Loader<VL>::load(gq[k], a.values + n * a.Ms + x0);
            Vec8Loader<VL>::load(aq[k], node_ptr(sa, n));
            Vec8Loader<VL>::load(bq[k], node_ptr(sb, n));
        }
    }
    for (long long base = 0; base < len; base += CHAIN_LA) {
#pragma unroll
        for (int k = 0; k < CHAIN_LA; ++k) {
            const long long pos = base + k;
            if (pos >= len) break;   // warp-uniform: the chains of a warp have one length
            const long long src = src0 + pos * geo.step;
            if (j == 0 && pos + CHAIN_PF < len) {
                const long long pf = src + CHAIN_PF * geo.step;
                const unsigned bytes = (unsigned)(a.Ms * 4);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.values + pf * a.Ms), "r"(bytes) : "memory");
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(msgs + sa * S + (pf + W) * a.Ms), "r"(bytes) : "memory");
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(msgs + sb * S + (pf + W) * a.Ms), "r"(bytes) : "memory");
            }
            // included slots in ascending order for each pass:
            //   0 (excl 2, chain 1): m0 m1 m3 = a, chain, b
            //   1 (excl 1, chain 2): m0 m2 m3 = a, chain, b
            //   2 (excl 3, chain 0): m0 m1 m2 = chain, a, b
            //   3 (excl 0, chain 3): m1 m2 m3 = a, b, chain
            float h[VL];
            if (dir <= 1) chain_h<DOM, VL, LP>(gq[k], aq[k], chain, bq[k], dir, h);
            else if (dir == 2) chain_h<DOM, VL, LP>(gq[k], chain, aq[k], bq[k], dir, h);
            else chain_h<DOM, VL, LP>(gq[k], aq[k], bq[k], chain, dir, h);
            // refill this ring slot with the node CHAIN_LA steps ahead
            if (pos + CHAIN_LA < len) {
                const long long n = src + CHAIN_LA * geo.step;
                Vec8Loader<VL>::load(gq[k], a.values + n * a.Ms + x0);
                Vec8Loader<VL>::load(aq[k], node_ptr(sa, n));
                Vec8Loader<VL>::load(bq[k], node_ptr(sb, n));
            }
            bool ok;
            if (dir == 0 || dir == 2) ok = band_message<DOM, VL, LP, R, 0>(a, h, j, x0, chain);
            else ok = band_message<DOM, VL, LP, R, 1>(a, h, j, x0, chain);
            if (a.delta && valid)
                dmax = fmaxf(dmax, message_delta<DOM, VL>(chain, node_ptr(geo.wslot, src + geo.step),
                                                          false, x0, a.M));
            if (valid) Vec8Loader<VL>::store(node_ptr(geo.wslot, src + geo.step), chain);
            if (!ok && valid && j == 0) {
                // reference order of the first failure: sweep, pass, line, position
                const unsigned long long key = ((unsigned long long)a.iteration << 40) |
                                               ((unsigned long long)dir << 38) |
                                               (unsigned long long)(line * len + pos);
                atomicMin(a.err, key);
            }
        }
    }
    if (a.delta) flush_delta(a.delta, dmax);
}

template <int DOM, int VL, int LP, int R>
cudaError_t launch_chain(const BandArgs &a, cudaStream_t s) {
    for (int dir = 0; dir < 4; ++dir) {
        BandArgs b = a;
        b.pass = dir;
        const long long lines = dir <= 1 ? a.H : a.W;
        const long long len = dir <= 1 ? a.W - 1 : a.H - 1;
        if (len <= 0) continue;
        const long long threads = lines * LP;
        const long long blocks = (threads + 127) / 128;
        chain_pass_kernel<DOM, VL, LP, R><<<(unsigned)blocks, 128, 0, s>>>(b);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <int MS, int DOM>
BandLaunchFn pick_chain(int R, int vl) {
    switch (R) {
#define SBP_CASE(RR)                                                         \
    case RR:                                                                 \
        if constexpr (RR < MS) {                                             \
            if constexpr (DOM == SBP_SUM && MS >= 128 && RR <= 8)            \
                if (vl == 16) return &launch_chain<DOM, 16, MS / 16, RR>;    \
            return &launch_chain<DOM, 8, MS / 8, RR>;                        \
        }                                                                    \
        return nullptr;
        SBP_BAND_RADII(SBP_CASE)
#undef SBP_CASE
    default: return nullptr;
    }
}

}  // namespace sbp
