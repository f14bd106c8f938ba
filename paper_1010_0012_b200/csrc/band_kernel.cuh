// Fused synchronous banded BP iteration (sm_100a).
//
// One launch performs every directed message update of a row range for one
// synchronous iteration.  Per node it reads the unary and the four incoming
// messages ONCE (256-bit loads, label-contiguous [slot][row][W][Ms] layout),
// forms the four exclusion products h_{i\j} in registers, and for each
// outgoing direction computes the reference "fast" update
//     sum:  out[x_j] = fbar * sum_x h(x) + sum_{d=-R..R} res(d) h(x_j + d)
//     max:  out[x_j] = max(fbar + max_x h(x), max_d (val(d) + h(x_j + d)))
// (numba_kernels.py:44-54 / 77-90, Eq. 7 / Eq. 11 of the paper) followed by
// the reference normalisation (numba_kernels.py:248-271) and a 256-bit store
// into the neighbour's incoming slot.
//
// Thread mapping: LP lanes own one node (pixel), each lane VL consecutive
// labels (VL*LP = Ms).  Sums/maxima over labels are in-lane then xor
// butterflies across the LP lanes (identical in every lane); the band's
// out-of-lane neighbours h(x +- s) come from __shfl_up/down of the owning
// lane.  The band is streamed in ascending x_i so every output accumulates its
// terms in the reference's order (ascending x_i over the stored column).
// Band weights depend only on d = x_i - x_j (Toeplitz potentials such as the
// truncated linear / quadratic families); they are kernel parameters, so
// every FFMA reads its weight straight from the constant bank.
#pragma once

#include "sbp_common.cuh"

#ifndef SBP_L1NA
#define SBP_L1NA 0   // 1: streaming loads / stores skip L1 allocation
#endif
#if SBP_L1NA
#define SBP_L1_HINT ".L1::no_allocate"
#else
#define SBP_L1_HINT ""
#endif

#ifndef SBP_HSMEM
#define SBP_HSMEM 0   // 1: out-of-lane band taps through shared memory (measured slower, profiles/r01_ab_hsmem.txt)
#endif

namespace sbp {

struct BandArgs {
    const float *values;   // [rows][W][Ms]
    const float *msgs_in;  // [4][rows+2][W][Ms]
    float *msgs_out;
    unsigned long long *err;
    long long slot_stride;  // (rows+2)*W*Ms
    int H, W, M, Ms, r0, lr_begin, lr_end, iteration, floor_term;
    int first;   // iteration 0: incoming messages are the reference init, not read
    int pass;      // sequential mode: pass direction 0..3 (chain_kernel.cuh)
    float fbar[2];
    float w[2][2 * SBP_MAX_R + 1];
    // Pair table for the packed band: wp[o][k] = (w(k-R-1), w(k-R-2)), with
    // w(d) = pad (0 / -inf) for |d| > R, R the compiled radius (band_pairs()).
    float2 wp[2][2 * SBP_MAX_R + 4];
    // Fused convergence test (bp.py:671-676): when set, every written message
    // also compares itself with the value it replaces in the previous
    // iteration's buffer (the same slot of msgs_in; in place for sweeps) and
    // the kernel max-reduces |new - old| into *delta (non-negative floats
    // compare as ints: atomicMax on the bits).  NULL: off.
    float *delta;
};

// Fills BandArgs::wp from BandArgs::w for the compiled radius R.
__host__ inline void band_pairs(BandArgs &a, int R, float pad) {
    for (int o = 0; o < 2; ++o)
        for (int k = 0; k < 2 * SBP_MAX_R + 4; ++k) {
            const int d0 = k - R - 1, d1 = k - R - 2;
            a.wp[o][k].x = (d0 >= -R && d0 <= R) ? a.w[o][d0 + R] : pad;
            a.wp[o][k].y = (d1 >= -R && d1 <= R) ? a.w[o][d1 + R] : pad;
        }
}

// Per-iteration view of the buffers: which buffer is read / written, the
// first row of the range, the iteration index (error key) and whether the
// incoming messages are the initial ones.  The plain kernels build it from
// BandArgs; the wavefront kernel changes it per work item.
struct IterCtx {
    const float *msgs_in;
    float *msgs_out;
    int lr_begin, iteration, first;
    float *dmax;   // this thread's running max |new - old| (BandArgs::delta)
};

__device__ __forceinline__ IterCtx iter_of(const BandArgs &a, float *dmax = nullptr) {
    return IterCtx{a.msgs_in, a.msgs_out, a.lr_begin, a.iteration, a.first, dmax};
}

// Largest |out - old| over a lane's labels, old = the message this one
// replaces (iteration 0: the reference initial message, bp.py:587-601).
// Padded labels give 0 (sum: 0 - 0) or NaN (max: -inf - -inf), which fmaxf
// drops.  `src` points at the old value (plain load: in place for sweeps).
template <int DOM, int VL>
__device__ __forceinline__ float message_delta(const float (&out)[VL], const float *src,
                                               bool first, int x0, int M) {
    float old[VL];
    if (first) {
#pragma unroll
        for (int i = 0; i < VL; ++i)
            old[i] = x0 + i < M ? (DOM == SBP_SUM ? 1.0f / (float)M : 0.0f) : out[i];
    } else {
#pragma unroll
        for (int c = 0; c < VL / 8; ++c) {
            const float *p = src + 8 * c;
            asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(old[8 * c + 0]), "=f"(old[8 * c + 1]), "=f"(old[8 * c + 2]),
                           "=f"(old[8 * c + 3]), "=f"(old[8 * c + 4]), "=f"(old[8 * c + 5]),
                           "=f"(old[8 * c + 6]), "=f"(old[8 * c + 7])
                         : "l"(p));
        }
    }
    float d = 0.0f;
#pragma unroll
    for (int i = 0; i < VL; ++i) d = fmaxf(d, fabsf(out[i] - old[i]));
    return d;
}

// End of a delta-enabled launch: one atomic per warp.
__device__ __forceinline__ void flush_delta(float *delta, float dmax) {
#pragma unroll
    for (int off = 16; off; off >>= 1) dmax = fmaxf(dmax, __shfl_xor_sync(SBP_FULL_MASK, dmax, off));
    if ((threadIdx.x & 31) == 0 && dmax > 0.0f) atomicMax(reinterpret_cast<int *>(delta), __float_as_int(dmax));
}

template <int N>
struct Vec8Loader {
    static __device__ __forceinline__ void load(float (&dst)[N], const float *src) {
#pragma unroll
        for (int c = 0; c < N / 8; ++c) {
            const float *p = src + 8 * c;
            asm volatile(
                "ld.global.nc" SBP_L1_HINT ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=f"(dst[8 * c + 0]), "=f"(dst[8 * c + 1]), "=f"(dst[8 * c + 2]),
                  "=f"(dst[8 * c + 3]), "=f"(dst[8 * c + 4]), "=f"(dst[8 * c + 5]),
                  "=f"(dst[8 * c + 6]), "=f"(dst[8 * c + 7])
                : "l"(p));
        }
    }
    static __device__ __forceinline__ void store(float *dst, const float (&v)[N]) {
#pragma unroll
        for (int c = 0; c < N / 8; ++c) {
            float *p = dst + 8 * c;
            asm volatile("st.global" SBP_L1_HINT ".v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                         "f"(v[8 * c + 0]), "f"(v[8 * c + 1]), "f"(v[8 * c + 2]),
                         "f"(v[8 * c + 3]), "f"(v[8 * c + 4]), "f"(v[8 * c + 5]),
                         "f"(v[8 * c + 6]), "f"(v[8 * c + 7])
                         : "memory");
        }
    }
};

template <int LP>
__device__ __forceinline__ float lanes_sum(float v) {
#pragma unroll
    for (int off = 1; off < LP; off <<= 1) v += __shfl_xor_sync(SBP_FULL_MASK, v, off);
    return v;
}

// RX: the warp-wide float max of sm_100a in one instruction (redux.sync.max.f32,
// SASS CREDUX.MAX.F32; NaN operands are ignored like fmaxf) instead of five
// SHFL + FMNMX steps.  Same value, so same bits; opt-in per kernel (it wins
// for the max-sum tap kernels at R <= 16: C5 T=9 2.05 -> 1.92 ms, T=17 2.78 ->
// 2.65, and loses 2 % in the one-copy R = 32 body; profiles/r02_ab_redux.txt).
template <int LP, bool RX = false>
__device__ __forceinline__ float lanes_max(float v) {
    if (RX && LP == 32) {
        float r;
        asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
        return r;
    }
#pragma unroll
    for (int off = 1; off < LP; off <<= 1) v = fmaxf(v, __shfl_xor_sync(SBP_FULL_MASK, v, off));
    return v;
}

// Kernels whose warp-wide maxima use redux.sync (lanes_max RX): max-sum, one
// node per warp (Ms = 256), 4 <= R <= 16 -- measured per C5 band: T=5 1.86 ->
// 1.61 ms, T=9 2.05 -> 1.92, T=17 2.78 -> 2.65; slower for R = 1 (T=2: 1.55 ->
// 1.68) and in the one-copy R = 32 body (profiles/r02_ab_redux.txt).
template <int DOM, int LP, int R>
constexpr bool band_redux() { return DOM == SBP_MAX && LP == 32 && R >= 4 && R <= 16; }

// h value at lane-relative label offset t (t in [-R, VL+R)).
template <int DOM, int VL, int LP, int R>
__device__ __forceinline__ float band_h(const float (&h)[VL], int t, int j) {
    constexpr float PAD = DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    if (t >= 0 && t < VL) return h[t];
    if (t < 0) {
        const int s = -t;
        const int q = (s + VL - 1) / VL;
        if (q >= LP) return PAD;
        const int idx = q * VL - s;
        float v = __shfl_up_sync(SBP_FULL_MASK, h[idx], q, LP);
        return j >= q ? v : PAD;
    }
    const int s = t - VL + 1;
    const int q = (s + VL - 1) / VL;
    if (q >= LP) return PAD;
    const int idx = s - 1 - (q - 1) * VL;
    float v = __shfl_down_sync(SBP_FULL_MASK, h[idx], q, LP);
    return j + q < LP ? v : PAD;
}

// The band's out-of-lane taps h(x0 + t), t in [-R, 0) and [VL, VL + R): the
// neighbouring lanes' labels of the same node, or the pad (0 / -inf) past
// the node's first / last label.  SBP_HSMEM: every lane stores its h into a
// per-node shared-memory row [pad | h(Ms) | pad] and reads its taps back with
// 128-bit loads (2 * ceil(R/4) LDS.128 instead of 2R shuffles + selects),
// for R >= 5.
// Blocks are 4 warps (every kernel that calls band_message launches 128
// threads); the row of a node is private to its warp.
template <int DOM, int VL, int LP, int R>
struct BandTaps {
    static constexpr int RL = (R + 3) / 4 * 4;   // floats fetched per side
    float lo[RL], hi[RL];

    __device__ __forceinline__ void fetch(const float (&h)[VL], int j, int x0) {
        // narrow bands keep the shuffles (fewer instructions at R <= 4 in SASS)
        if constexpr (SBP_HSMEM && R >= 5) {
        constexpr int PPW = 32 / LP, MS = VL * LP, PADF = RL < 4 ? 4 : RL;
        constexpr int ROW = MS + 2 * PADF;
        constexpr float PAD = DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf();
        __shared__ __align__(16) float hsm[4 * PPW * ROW];
        float *row = hsm + ((threadIdx.x >> 5) * PPW + (threadIdx.x & 31) / LP) * ROW;
        __syncwarp();   // the previous message's reads of this row are done
#pragma unroll
        for (int i = 0; i < VL; i += 4)
            *reinterpret_cast<float4 *>(row + PADF + x0 + i) = make_float4(h[i], h[i + 1], h[i + 2], h[i + 3]);
        if (j == 0) {
#pragma unroll
            for (int i = 0; i < PADF; i += 4) *reinterpret_cast<float4 *>(row + i) = make_float4(PAD, PAD, PAD, PAD);
        }
        if (j == LP - 1) {
#pragma unroll
            for (int i = 0; i < PADF; i += 4)
                *reinterpret_cast<float4 *>(row + PADF + MS + i) = make_float4(PAD, PAD, PAD, PAD);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < RL; i += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(row + PADF + x0 - RL + i);
            lo[i] = v.x; lo[i + 1] = v.y; lo[i + 2] = v.z; lo[i + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < RL; i += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(row + PADF + x0 + VL + i);
            hi[i] = v.x; hi[i + 1] = v.y; hi[i + 2] = v.z; hi[i + 3] = v.w;
        }
        } else {
#pragma unroll
        for (int t = -R; t < 0; ++t) lo[RL + t] = band_h<DOM, VL, LP, R>(h, t, j);
#pragma unroll
        for (int t = VL; t < VL + R; ++t) hi[t - VL] = band_h<DOM, VL, LP, R>(h, t, j);
        }
    }

    __device__ __forceinline__ float at(const float (&h)[VL], int t) const {
        return t < 0 ? lo[RL + t] : (t < VL ? h[t] : hi[t - VL]);
    }
};

// Three-input max (sm_100 FMNMX3): exact, same NaN rule as fmaxf.
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Knuth TwoSum: a + b = s + e exactly (no FMA contraction: adds only).
// With -inf operands (log of a zero unary / potential entry, label padding)
// e becomes NaN; once a partial sum is -inf it stays -inf (there is no +inf),
// so the NaN is discarded once, on the final sum, in shift_compensated.
__device__ __forceinline__ void two_sum(float a, float b, float &s, float &e) {
    s = a + b;
    const float bp = s - a;
    e = (a - (s - bp)) + (b - bp);
}

// h'[i] = (s[i] - c) + e[i] with c = max over the node's labels of s.
// Pairs of labels use the packed FP32 ops (bit-identical to the scalar ones).
template <int VL, int LP, bool RX = false>
__device__ __forceinline__ void shift_compensated(const float (&s)[VL], const float (&e)[VL],
                                                  float (&h)[VL]) {
    float c = s[0];
    int i0 = 1;
    if (VL % 2 == 0 && VL > 1) { c = fmaxf(s[0], s[1]); i0 = 2; }
#pragma unroll
    for (int i = i0; i + 1 < VL; i += 2) c = fmax3(c, s[i], s[i + 1]);
    if ((VL - i0) % 2 == 1) c = fmaxf(c, s[VL - 1]);
    c = lanes_max<LP, RX>(c);
    if (!isfinite(c)) c = 0.0f;
#pragma unroll
    for (int i = 0; i + 1 < VL; i += 2) {
        float d0, d1;
        sub2(d0, d1, s[i], s[i + 1], c, c);
        add2(h[i], h[i + 1], d0, d1, isfinite(s[i]) ? e[i] : 0.0f,
             isfinite(s[i + 1]) ? e[i + 1] : 0.0f);
    }
    if (VL % 2 == 1) h[VL - 1] = (s[VL - 1] - c) + (isfinite(s[VL - 1]) ? e[VL - 1] : 0.0f);
}

// Sum of a lane's VL labels: even and odd labels accumulate in the two halves
// of a packed pair (FADD2), then combine -- half the instructions and half
// the dependent-add chain of a serial sum.
template <int VL>
__device__ __forceinline__ float vsum(const float (&v)[VL]) {
    float s0 = v[0], s1 = v[1];
#pragma unroll
    for (int i = 2; i < VL; i += 2) add2(s0, s1, s0, s1, v[i], v[i + 1]);
    return s0 + s1;
}

// Pairwise helpers over VL-label arrays (VL even).
template <int VL>
__device__ __forceinline__ void vmul(float (&r)[VL], const float (&a)[VL], const float (&b)[VL]) {
#pragma unroll
    for (int i = 0; i < VL; i += 2) mul2(r[i], r[i + 1], a[i], a[i + 1], b[i], b[i + 1]);
}

// (s, e) = TwoSum(a, b) label-wise
template <int VL>
__device__ __forceinline__ void vtwo_sum(const float (&a)[VL], const float (&b)[VL], float (&s)[VL],
                                         float (&e)[VL]) {
#pragma unroll
    for (int i = 0; i < VL; i += 2)
        two_sum2(a[i], a[i + 1], b[i], b[i + 1], s[i], s[i + 1], e[i], e[i + 1]);
}

// s += b error-free, the new error added to e0 into e: (s, e) = (s + b, e0 + err)
template <int VL>
__device__ __forceinline__ void vtwo_sum_acc(float (&s)[VL], const float (&b)[VL],
                                             const float (&e0)[VL], float (&e)[VL]) {
#pragma unroll
    for (int i = 0; i < VL; i += 2) {
        float t0, t1, x0, x1;
        two_sum2(s[i], s[i + 1], b[i], b[i + 1], t0, t1, x0, x1);
        s[i] = t0; s[i + 1] = t1;
        add2(e[i], e[i + 1], e0[i], e0[i + 1], x0, x1);
    }
}

// (s, e) = TwoSum(a, b) with e = e0 + err (a fresh sum from a prefix a + e0)
template <int VL>
__device__ __forceinline__ void vtwo_sum_from(const float (&a)[VL], const float (&e0)[VL],
                                              const float (&b)[VL], float (&s)[VL], float (&e)[VL]) {
#pragma unroll
    for (int i = 0; i < VL; i += 2) {
        float x0, x1;
        two_sum2(a[i], a[i + 1], b[i], b[i + 1], s[i], s[i + 1], x0, x1);
        add2(e[i], e[i + 1], e0[i], e0[i + 1], x0, x1);
    }
}

// One outgoing direction: fast update + normalisation + store.
// O (orientation) is compile-time so every weight is a constant-bank operand;
// DIR is a compile-time constant in the unrolled kernel and a runtime value in
// the rolled one (store slot / step / edge id only).
// The message of one directed edge from its exclusion vector h: the fast
// update (floor term + band) and the reference normalisation.  Returns
// whether the message could be normalised.
template <int DOM, int VL, int LP, int R, int O>
__device__ __forceinline__ bool band_message(const BandArgs &a, const float (&h)[VL], int j,
                                             int x0, float (&out)[VL]) {
    if (DOM == SBP_SUM) {
        const float s = lanes_sum<LP>(vsum(h));
        const float base = a.floor_term ? a.fbar[O] * s : 0.0f;
#pragma unroll
        for (int i = 0; i < VL; ++i) out[i] = base;
    } else {
        float mx = fmaxf(h[0], h[1]);
#pragma unroll
        for (int i = 2; i < VL; i += 2) mx = fmax3(mx, h[i], h[i + 1]);
        mx = lanes_max<LP, band_redux<DOM, LP, R>()>(mx);
        const float base = a.floor_term ? a.fbar[O] + mx : -__builtin_huge_valf();
#pragma unroll
        for (int i = 0; i < VL; ++i) out[i] = base;
    }
    // Band, streamed in ascending x_i: term (x_i = x0+t) reaches out[i] at d = t - i.
    // Label pairs (out[i], out[i+1]) take the weights (w(d), w(d-1)) of the
    // pair table in one packed op; taps outside |d| <= R carry the pad weight
    // (0 / -inf), exact no-ops, so every pair op is unconditional.
    BandTaps<DOM, VL, LP, R> taps;
    taps.fetch(h, j, x0);
    if (DOM == SBP_SUM) {
#pragma unroll
        for (int t = -R; t < VL + R; ++t) {
            const float hv = taps.at(h, t);
#pragma unroll
            for (int i = 0; i < VL; i += 2) {
                const int d = t - i;
                if (d < -R || d > R + 1) continue;
                fma2(out[i], out[i + 1], a.wp[O][d + R + 1], hv);
            }
        }
    } else {
        // two taps per FMNMX3 (the max is exact: any grouping gives the same bits)
#pragma unroll
        for (int t = -R; t < VL + R; t += 2) {
            const bool has1 = t + 1 < VL + R;
            const float hv0 = taps.at(h, t);
            const float hv1 = has1 ? taps.at(h, t + 1) : 0.0f;
#pragma unroll
            for (int i = 0; i < VL; i += 2) {
                const int d0 = t - i, d1 = t + 1 - i;
                const bool in0 = d0 >= -R && d0 <= R + 1;
                const bool in1 = has1 && d1 >= -R && d1 <= R + 1;
                float a0, a1, b0, b1;
                if (in0) add2(a0, a1, a.wp[O][d0 + R + 1].x, a.wp[O][d0 + R + 1].y, hv0, hv0);
                if (in1) add2(b0, b1, a.wp[O][d1 + R + 1].x, a.wp[O][d1 + R + 1].y, hv1, hv1);
                if (in0 && in1) {
                    out[i] = fmax3(out[i], a0, b0);
                    out[i + 1] = fmax3(out[i + 1], a1, b1);
                } else if (in0) {
                    out[i] = fmaxf(out[i], a0);
                    out[i + 1] = fmaxf(out[i + 1], a1);
                } else if (in1) {
                    out[i] = fmaxf(out[i], b0);
                    out[i + 1] = fmaxf(out[i + 1], b1);
                }
            }
        }
    }
    // Normalise (numba_kernels.py:248-271); padded labels stay 0 / -inf.
    bool ok;
    if (DOM == SBP_SUM) {
        if (a.M < a.Ms) {
#pragma unroll
            for (int i = 0; i < VL; ++i)
                if (x0 + i >= a.M) out[i] = 0.0f;
        }
        const float s = lanes_sum<LP>(vsum(out));
        ok = (s > 0.0f) && !isinf(s);
        const float inv = __frcp_rn(s);
#pragma unroll
        for (int i = 0; i < VL; i += 2) mul2(out[i], out[i + 1], out[i], out[i + 1], inv, inv);
    } else {
        if (a.M < a.Ms) {
#pragma unroll
            for (int i = 0; i < VL; ++i)
                if (x0 + i >= a.M) out[i] = -__builtin_huge_valf();
        }
        float mx = fmaxf(out[0], out[1]);
#pragma unroll
        for (int i = 2; i < VL; i += 2) mx = fmax3(mx, out[i], out[i + 1]);
        mx = lanes_max<LP, band_redux<DOM, LP, R>()>(mx);
        ok = isfinite(mx);
#pragma unroll
        for (int i = 0; i < VL; i += 2) sub2(out[i], out[i + 1], out[i], out[i + 1], mx, mx);
    }
    return ok;
}

template <int DOM, int VL, int LP, int R, int O>
__device__ __forceinline__ void emit_direction(const BandArgs &a, const IterCtx &it,
                                               const float (&h)[VL], int DIR, int j, int x0,
                                               bool active, long long node_l, long long r,
                                               int c) {
    float out[VL];
    const bool ok = band_message<DOM, VL, LP, R, O>(a, h, j, x0, out);
    if (!active) return;
    const long long W = a.W;
    // node part (loop-invariant in the rolled kernel) + a warp-uniform
    // direction offset: slot of the neighbour and the step to it
    const long long step = DIR == 0 ? 1 : DIR == 1 ? -1 : DIR == 2 ? W : -W;
    const long long dir_off = dir_wslot(DIR) * a.slot_stride + step * a.Ms;
    float *dst = it.msgs_out + (node_l * a.Ms + x0) + dir_off;
    if (a.delta)
        *it.dmax = fmaxf(*it.dmax, message_delta<DOM, VL>(out, it.msgs_in + (node_l * a.Ms + x0) + dir_off,
                                                         it.first, x0, a.M));
    Vec8Loader<VL>::store(dst, out);
    if (!ok && j == 0) report_failure(a.err, it.iteration, directed_edge_id(a.H, W, r, c, DIR));
}

// The four messages of one node from its unary and incoming vectors.
template <int DOM, int VL, int LP, int R>
__device__ __forceinline__ void band_group_body(const BandArgs &a, const IterCtx &it,
                                                const float (&g)[VL],
                                                const float (&m0)[VL], const float (&m1)[VL],
                                                const float (&m2)[VL], const float (&m3)[VL],
                                                int j, int x0, bool valid, long long node_l,
                                                long long r, int c) {
    const bool has_r = c + 1 < a.W, has_l = c > 0, has_d = r + 1 < a.H, has_u = r > 0;
    float h[VL];
    if (DOM == SBP_SUM) {
        // Exclusion products in the reference order: unary, then slots 0..3
        // ascending, skipping the excluded one (numba_kernels.py:194-227).
        float ab[VL];
        vmul(ab, g, m0);                                                     // g m0
        if (__any_sync(SBP_FULL_MASK, valid && has_u)) {                     // excl 0
            vmul(h, g, m1);
            vmul(h, h, m2);
            vmul(h, h, m3);
            emit_direction<DOM, VL, LP, R, dir_orient(3)>(a, it, h, 3, j, x0, valid && has_u, node_l, r, c);
        }
        if (__any_sync(SBP_FULL_MASK, valid && has_l)) {                     // excl 1
            vmul(h, ab, m2);
            vmul(h, h, m3);
            emit_direction<DOM, VL, LP, R, dir_orient(1)>(a, it, h, 1, j, x0, valid && has_l, node_l, r, c);
        }
        vmul(ab, ab, m1);                                                    // g m0 m1
        if (__any_sync(SBP_FULL_MASK, valid && has_r)) {                     // excl 2
            vmul(h, ab, m3);
            emit_direction<DOM, VL, LP, R, dir_orient(0)>(a, it, h, 0, j, x0, valid && has_r, node_l, r, c);
        }
        if (__any_sync(SBP_FULL_MASK, valid && has_d)) {                     // excl 3
            vmul(h, ab, m2);
            emit_direction<DOM, VL, LP, R, dir_orient(2)>(a, it, h, 2, j, x0, valid && has_d, node_l, r, c);
        }
    } else {
        // Max-sum: h = ln g + sum of three messages.  Its entries can reach
        // tens in magnitude while the normalised messages resolve ~1e-7, so
        // fp32 rounding of the sum dominates the error (measured: 8.5e-6 on
        // C5 T=9).  The sum is formed error-free (TwoSum: h = s + e exactly
        // up to ~2^-48 relative), shifted by the node's max of s, and only
        // then rounded: h' = (s - c) + e.  Messages are shift-invariant.
        float sa[VL], ea[VL], s2[VL], e2[VL];
        vtwo_sum(g, m0, sa, ea);                                             // g + m0
        if (__any_sync(SBP_FULL_MASK, valid && has_u)) {                     // excl 0
            vtwo_sum(g, m1, s2, e2);
            vtwo_sum_acc(s2, m2, e2, e2);
            vtwo_sum_acc(s2, m3, e2, e2);
            shift_compensated<VL, LP, band_redux<DOM, LP, R>()>(s2, e2, h);
            emit_direction<DOM, VL, LP, R, dir_orient(3)>(a, it, h, 3, j, x0, valid && has_u, node_l, r, c);
        }
        if (__any_sync(SBP_FULL_MASK, valid && has_l)) {                     // excl 1
            vtwo_sum_from(sa, ea, m2, s2, e2);
            vtwo_sum_acc(s2, m3, e2, e2);
            shift_compensated<VL, LP, band_redux<DOM, LP, R>()>(s2, e2, h);
            emit_direction<DOM, VL, LP, R, dir_orient(1)>(a, it, h, 1, j, x0, valid && has_l, node_l, r, c);
        }
        vtwo_sum_acc(sa, m1, ea, ea);                                        // g + m0 + m1
        if (__any_sync(SBP_FULL_MASK, valid && has_r)) {                     // excl 2
            vtwo_sum_from(sa, ea, m3, s2, e2);
            shift_compensated<VL, LP, band_redux<DOM, LP, R>()>(s2, e2, h);
            emit_direction<DOM, VL, LP, R, dir_orient(0)>(a, it, h, 0, j, x0, valid && has_r, node_l, r, c);
        }
        if (__any_sync(SBP_FULL_MASK, valid && has_d)) {                     // excl 3
            vtwo_sum_from(sa, ea, m2, s2, e2);
            shift_compensated<VL, LP, band_redux<DOM, LP, R>()>(s2, e2, h);
            emit_direction<DOM, VL, LP, R, dir_orient(2)>(a, it, h, 2, j, x0, valid && has_d, node_l, r, c);
        }
    }
}

// One warp-group of PPW = 32/LP nodes (flattened pixel group `grp`).
template <int DOM, int VL, int LP, int R>
__device__ __forceinline__ void band_group(const BandArgs &a, const IterCtx &it, long long grp,
                                   long long npix) {
    constexpr int PPW = 32 / LP;
    const int lane = threadIdx.x & 31;
    const int j = lane % LP;
    long long p = grp * PPW + lane / LP;
    const bool valid = p < npix;
    if (!valid) p = npix - 1;
    const int lr = it.lr_begin + (int)(p / a.W);
    const int c = (int)(p % a.W);
    const long long r = (long long)a.r0 + lr - 1;
    const long long node_l = (long long)lr * a.W + c;
    const int x0 = j * VL;

    float g[VL], m0[VL], m1[VL], m2[VL], m3[VL];
    Vec8Loader<VL>::load(g, a.values + ((long long)(lr - 1) * a.W + c) * a.Ms + x0);
    const float *mi = it.msgs_in + node_l * a.Ms + x0;
    if (!it.first) {
        Vec8Loader<VL>::load(m0, mi);
        Vec8Loader<VL>::load(m1, mi + a.slot_stride);
        Vec8Loader<VL>::load(m2, mi + 2 * a.slot_stride);
        Vec8Loader<VL>::load(m3, mi + 3 * a.slot_stride);
    } else {
        // bp.py:587-601 without touching memory: 1/M on real slots, the
        // identity on ghost slots, padding 0 / -inf
        const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
        float *mm[4] = {m0, m1, m2, m3};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float real = DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M) : 0.0f;
#pragma unroll
            for (int i = 0; i < VL; ++i)
                mm[k][i] = x0 + i < a.M ? real : (DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf());
        }
    }

    band_group_body<DOM, VL, LP, R>(a, it, g, m0, m1, m2, m3, j, x0, valid, node_l, r, c);
}

template <int DOM, int VL, int LP, int R>
__device__ __forceinline__ void band_group_body_rolled(const BandArgs &a, const IterCtx &it,
                                                       const float (&g)[VL],
                                                       const float (&m0)[VL], const float (&m1)[VL],
                                                       const float (&m2)[VL], const float (&m3)[VL],
                                                       int j, int x0, bool valid, long long node_l,
                                                       long long r, int c);

// Rolled variant for potentials whose two orientations carry the same band
// (symmetric f, e.g. every truncated-linear / quadratic config): one copy of
// the fully unrolled band serves all four directions (runtime loop), cutting
// the instruction footprint 4x -- the unrolled kernel spills the I-cache for
// wide bands (ncu: 34 % of issue slots lost to instruction fetch at R = 32).
template <int DOM, int VL, int LP, int R>
__device__ __forceinline__ void band_group_rolled(const BandArgs &a, const IterCtx &it, long long grp,
                                   long long npix) {
    constexpr int PPW = 32 / LP;
    const int lane = threadIdx.x & 31;
    const int j = lane % LP;
    long long p = grp * PPW + lane / LP;
    const bool valid = p < npix;
    if (!valid) p = npix - 1;
    const int lr = it.lr_begin + (int)(p / a.W);
    const int c = (int)(p % a.W);
    const long long r = (long long)a.r0 + lr - 1;
    const long long node_l = (long long)lr * a.W + c;
    const int x0 = j * VL;

    float g[VL], m0[VL], m1[VL], m2[VL], m3[VL];
    Vec8Loader<VL>::load(g, a.values + ((long long)(lr - 1) * a.W + c) * a.Ms + x0);
    const float *mi = it.msgs_in + node_l * a.Ms + x0;
    if (!it.first) {
        Vec8Loader<VL>::load(m0, mi);
        Vec8Loader<VL>::load(m1, mi + a.slot_stride);
        Vec8Loader<VL>::load(m2, mi + 2 * a.slot_stride);
        Vec8Loader<VL>::load(m3, mi + 3 * a.slot_stride);
    } else {
        const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
        float *mm[4] = {m0, m1, m2, m3};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float real = DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M) : 0.0f;
#pragma unroll
            for (int i = 0; i < VL; ++i)
                mm[k][i] = x0 + i < a.M ? real : (DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf());
        }
    }
    band_group_body_rolled<DOM, VL, LP, R>(a, it, g, m0, m1, m2, m3, j, x0, valid, node_l, r, c);
}

// The four messages of one node, one band copy for all four directions.
template <int DOM, int VL, int LP, int R>
__device__ __forceinline__ void band_group_body_rolled(const BandArgs &a, const IterCtx &it,
                                                       const float (&g)[VL],
                                                       const float (&m0)[VL], const float (&m1)[VL],
                                                       const float (&m2)[VL], const float (&m3)[VL],
                                                       int j, int x0, bool valid, long long node_l,
                                                       long long r, int c) {
    // bit d: the node has a neighbour in direction d (no local arrays:
    // runtime-indexed arrays would live in local memory)
    const unsigned has = (c + 1 < a.W ? 1u : 0u) | (c > 0 ? 2u : 0u) |
                         (r + 1 < a.H ? 4u : 0u) | (r > 0 ? 8u : 0u);
    // prefixes shared by the directions (same association as the unrolled
    // kernel, so both variants give identical bits)
    float pa[VL], pb[VL], ea[VL], eb[VL];
    if (DOM == SBP_SUM) {
        vmul(pa, g, m0);
        vmul(pb, pa, m1);
    } else {
        vtwo_sum(g, m0, pa, ea);
        vtwo_sum_from(pa, ea, m1, pb, eb);
    }
#pragma unroll 1
    for (int k = 0; k < 4; ++k) {
        const int dir = (0x2013 >> (4 * k)) & 0xF;   // order 3, 1, 0, 2
        const bool hd = (has >> dir) & 1u;
        if (!__any_sync(SBP_FULL_MASK, valid && hd)) continue;
        float h[VL];
        if (DOM == SBP_SUM) {
            if (dir == 3) {
                vmul(h, g, m1);
                vmul(h, h, m2);
                vmul(h, h, m3);
            } else if (dir == 1) {
                vmul(h, pa, m2);
                vmul(h, h, m3);
            } else if (dir == 0) {
                vmul(h, pb, m3);
            } else {
                vmul(h, pb, m2);
            }
        } else {
            float s2[VL], e2[VL];
            if (dir == 3) {
                vtwo_sum(g, m1, s2, e2);
                vtwo_sum_acc(s2, m2, e2, e2);
                vtwo_sum_acc(s2, m3, e2, e2);
            } else if (dir == 1) {
                vtwo_sum_from(pa, ea, m2, s2, e2);
                vtwo_sum_acc(s2, m3, e2, e2);
            } else if (dir == 0) {
                vtwo_sum_from(pb, eb, m3, s2, e2);
            } else {
                vtwo_sum_from(pb, eb, m2, s2, e2);
            }
            shift_compensated<VL, LP, band_redux<DOM, LP, R>()>(s2, e2, h);
        }
        emit_direction<DOM, VL, LP, R, 0>(a, it, h, dir, j, x0, valid && hd, node_l, r, c);
    }
}

// ---------------------------------------------------------------------------
// TMA-staged variant: each warp double-buffers its pixel groups in shared
// memory with 1-D bulk copies (cp.async.bulk, completion on an mbarrier), so
// the next group's five input vectors are always in flight while the current
// one is computed -- memory-level parallelism without extra registers.
// ---------------------------------------------------------------------------
constexpr int STG_WARPS = 4;

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}

// NS = 2: double buffer, the next group's copy is issued before waiting for
// the current one.  NS = 1: one buffer, the next copy is issued as soon as the
// current group has moved to registers (half the shared memory, for VL = 16).
// Staged VL = 16 kernel (sum, Ms >= 128): 4 resident blocks per SM (124
// registers, no spills) instead of the 3 its 136 registers allowed: C5 T=5 sum
// 1.565 vs 1.595 ms per iteration, cold and sustained
// (profiles/r02_ab_staged16_blocks.txt).  0: no register bound.
#ifndef SBP_STG16_BLOCKS
#define SBP_STG16_BLOCKS 4
#endif
template <int DOM, int VL, int LP, int R, int NS>
__global__ void __launch_bounds__(32 * STG_WARPS, (VL == 16 ? SBP_STG16_BLOCKS : 0))
band_iter_staged_kernel(const __grid_constant__ BandArgs a) {
    constexpr int PPW = 32 / LP;
    float dmax = 0.0f;
    const IterCtx it = iter_of(a, &dmax);
    constexpr int VEC = 32 * VL;                 // floats of one vector for one group
    extern __shared__ __align__(128) float stg_smem[];
    __shared__ __align__(8) unsigned long long bars[STG_WARPS][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = lane % LP, q = lane / LP;
    const int x0 = j * VL;
    float *buf = stg_smem + warp * (NS * 5 * VEC);
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long ngroups = (npix + PPW - 1) / PPW;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (lane == 0) {
        mbar_init(&bars[warp][0], 1);
        mbar_init(&bars[warp][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int nvec = a.first ? 1 : 5;
    auto issue = [&](long long g, int st) {
        if (lane == 0) {
            const long long p0 = g * PPW;
            const long long n = npix - p0 < PPW ? npix - p0 : PPW;
            const unsigned bytes = (unsigned)(n * a.Ms * 4);
            float *dst = buf + st * 5 * VEC;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bars[warp][st], bytes * nvec);
            bulk_g2s(dst, a.values + ((long long)(a.lr_begin - 1) * a.W + p0) * a.Ms, bytes,
                     &bars[warp][st]);
            if (!a.first)
                for (int k = 0; k < 4; ++k)
                    bulk_g2s(dst + (1 + k) * VEC,
                             a.msgs_in + k * a.slot_stride + ((long long)a.lr_begin * a.W + p0) * a.Ms,
                             bytes, &bars[warp][st]);
        }
    };
    unsigned phase = 0;   // bit st: parity of stage st
    int st = 0;
    if (grp < ngroups) issue(grp, 0);
    for (; grp < ngroups; grp += nwarps) {
        if (NS == 2 && grp + nwarps < ngroups) issue(grp + nwarps, st ^ 1);
        mbar_wait(&bars[warp][st], (phase >> st) & 1);
        phase ^= 1u << st;
        long long p = grp * PPW + q;
        const bool valid = p < npix;
        if (!valid) p = npix - 1;
        const int lr = a.lr_begin + (int)(p / a.W);
        const int c = (int)(p % a.W);
        const long long r = (long long)a.r0 + lr - 1;
        const long long node_l = (long long)lr * a.W + c;
        const float *src = buf + st * 5 * VEC + q * a.Ms + x0;
        float g[VL], m0[VL], m1[VL], m2[VL], m3[VL];
#pragma unroll
        for (int i = 0; i < VL; i += 4) {
            const float4 v = *reinterpret_cast<const float4 *>(src + i);
            g[i] = v.x; g[i + 1] = v.y; g[i + 2] = v.z; g[i + 3] = v.w;
        }
        if (!a.first) {
            float *mm[4] = {m0, m1, m2, m3};
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int i = 0; i < VL; i += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(src + (1 + k) * VEC + i);
                    mm[k][i] = v.x; mm[k][i + 1] = v.y; mm[k][i + 2] = v.z; mm[k][i + 3] = v.w;
                }
        } else {
            const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
            float *mm[4] = {m0, m1, m2, m3};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float real = DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M) : 0.0f;
#pragma unroll
                for (int i = 0; i < VL; ++i)
                    mm[k][i] = x0 + i < a.M ? real : (DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf());
            }
        }
        __syncwarp();   // every lane has read stage st before it is refilled
        if (NS == 1 && grp + nwarps < ngroups) issue(grp + nwarps, 0);
        band_group_body<DOM, VL, LP, R>(a, it, g, m0, m1, m2, m3, j, x0, valid, node_l, r, c);
        if (NS == 2) st ^= 1;
    }
    if (a.delta) flush_delta(a.delta, dmax);
}

template <int DOM, int VL, int LP, int R, int NS>
cudaError_t launch_band_staged(const BandArgs &a, cudaStream_t s) {
    constexpr int PPW = 32 / LP;
    const size_t smem = (size_t)STG_WARPS * NS * 5 * 32 * VL * sizeof(float);
    static int resident = 0, sms = 0;
    if (!resident) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(band_iter_staged_kernel<DOM, VL, LP, R, NS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &resident, band_iter_staged_kernel<DOM, VL, LP, R, NS>, 32 * STG_WARPS, smem);
        if (resident < 1) resident = 1;
    }
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long warps = (npix + PPW - 1) / PPW;
    long long blocks = (warps + STG_WARPS - 1) / STG_WARPS;
    if (blocks <= 0) return cudaSuccess;
    const long long cap = (long long)sms * resident;
    if (blocks > cap) blocks = cap;
    if (launch_block_cap() > 0 && blocks > launch_block_cap()) blocks = launch_block_cap();
    band_iter_staged_kernel<DOM, VL, LP, R, NS><<<(unsigned)blocks, 32 * STG_WARPS, smem, s>>>(a);
    return cudaGetLastError();
}

// Persistent grid-stride kernel: each warp walks pixel groups grp, grp + T,
// ... (T = resident warps).  (An L2 prefetch of the next group measured
// slower on C4 and was dropped; the TMA-staged variant below is the
// latency-hiding version.)
#ifndef SBP_VL16_BLOCKS
#define SBP_VL16_BLOCKS 4   // resident 128-thread blocks per SM asked of ptxas for VL = 16, R <= 8
#endif
template <int DOM, int VL, int LP, int R, bool ROLLED>
__global__ void __launch_bounds__(128, (VL == 8 ? (DOM == SBP_SUM && R <= 7 ? 6 : 4) : (R <= 8 ? SBP_VL16_BLOCKS : 3)))
band_iter_kernel(const __grid_constant__ BandArgs a) {
    constexpr int PPW = 32 / LP;
    float dmax = 0.0f;
    const IterCtx it = iter_of(a, &dmax);
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long ngroups = (npix + PPW - 1) / PPW;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (; grp < ngroups; grp += nwarps) {
        if constexpr (ROLLED) band_group_rolled<DOM, VL, LP, R>(a, it, grp, npix);
        else band_group<DOM, VL, LP, R>(a, it, grp, npix);
    }
    if (a.delta) flush_delta(a.delta, dmax);
}

}  // namespace sbp

namespace sbp {

using BandLaunchFn = cudaError_t (*)(const BandArgs &, cudaStream_t);

template <int DOM, int VL, int LP, int R, bool ROLLED>
cudaError_t launch_band(const BandArgs &a, cudaStream_t s) {
    constexpr int PPW = 32 / LP;
    static int resident = 0;   // blocks of this instantiation per SM
    static int sms = 0;
    if (!resident) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &resident, band_iter_kernel<DOM, VL, LP, R, ROLLED>, 128, 0);
        if (resident < 1) resident = 1;
    }
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long warps = (npix + PPW - 1) / PPW;
    long long blocks = (warps + 3) / 4;
    if (blocks <= 0) return cudaSuccess;
    const long long cap = (long long)sms * resident;
    if (blocks > cap) blocks = cap;
    if (launch_block_cap() > 0 && blocks > launch_block_cap()) blocks = launch_block_cap();
    band_iter_kernel<DOM, VL, LP, R, ROLLED><<<(unsigned)blocks, 128, 0, s>>>(a);
    return cudaGetLastError();
}

// Band radii with a compiled kernel; a potential of radius r runs on the
// smallest listed R >= r (extra taps carry weight 0 / -inf: exact no-ops).
#define SBP_BAND_RADII(X) X(1) X(2) X(3) X(4) X(7) X(8) X(16) X(32)

template <int MS, int DOM, int VL, bool ROLLED>
BandLaunchFn pick_band_r(int R) {
    if constexpr (VL > MS) {
        return nullptr;
    } else {
        switch (R) {
#define SBP_CASE(RR)                                                      \
    case RR:                                                              \
        if constexpr (RR < MS && (!ROLLED || RR >= 24 || RR == 7 || RR == 8 || RR == 4) && \
                      (VL == 8 || ROLLED || RR <= 8))                         \
            return &launch_band<DOM, VL, MS / VL, RR, ROLLED>;             \
        else return nullptr;
            SBP_BAND_RADII(SBP_CASE)
#undef SBP_CASE
        default: return nullptr;
        }
    }
}

// VL = 16 is compiled only where the sweeps chose it (sum, Ms >= 128); the
// max domain always runs VL = 8 (its TwoSum state spills at VL = 16).
template <int MS, int DOM, int VL, int NS>
BandLaunchFn pick_band_staged_r(int R) {
    if constexpr (VL > MS) {
        return nullptr;
    } else {
        switch (R) {
#define SBP_CASE(RR)                                                      \
    case RR:                                                              \
        if constexpr (RR < MS && RR <= 16)                                \
            return &launch_band_staged<DOM, VL, MS / VL, RR, NS>;         \
        else return nullptr;
            SBP_BAND_RADII(SBP_CASE)
#undef SBP_CASE
        default: return nullptr;
        }
    }
}

// rolled: 0 unrolled, 1 rolled (symmetric, R >= 24), 2 TMA-staged unrolled (R <= 16)
template <int MS, int DOM>
BandLaunchFn pick_band_dom(int vl, int R, int rolled) {
    if (rolled == 2) {
        if (vl == 8) return pick_band_staged_r<MS, DOM, 8, 2>(R);
        if constexpr (DOM == SBP_SUM && MS >= 128)
            if (vl == 16) return pick_band_staged_r<MS, DOM, 16, 1>(R);
        return nullptr;
    }
    if (vl == 8) return rolled ? pick_band_r<MS, DOM, 8, true>(R) : pick_band_r<MS, DOM, 8, false>(R);
    if constexpr (DOM == SBP_SUM && MS >= 128) {
        if (vl == 16)
            return rolled ? pick_band_r<MS, DOM, 16, true>(R) : pick_band_r<MS, DOM, 16, false>(R);
    }
    return nullptr;
}

}  // namespace sbp
