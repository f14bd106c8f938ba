// General-potential iteration: per-column compatible lists in ELL form.
//
// Covers shared potentials that are not Toeplitz bands (arbitrary CSC, as
// produced by sparse_from_dense or the reference's random_sparse_potential,
// synth.py:21-43) and, with m_max = M and idx[k][x] = k, the reference's
// dense "standard" update (numba_kernels.py:35-41, 66-74).  One warp per
// node; h is staged in shared memory so the gather h[idx] is a broadcast /
// conflict-light LDS; entries of a column are visited in ascending x_i, the
// reference's order, padded entries carry weight 0 (sum) / -inf (max).
#include "aux_kernels.cuh"
#include "band_kernel.cuh"   // two_sum, shift_compensated, lanes_max

namespace sbp {

constexpr int ELL_WARPS = 4;
constexpr int ELL_QMAX = 8;   // Ms <= 256

template <int DOM, int DIR>
__device__ __forceinline__ void ell_emit(const EllArgs &a, const float (&h)[ELL_QMAX],
                                         float *hs, int lane, bool active, long long node_l,
                                         long long r, int c) {
    constexpr int O = dir_orient(DIR);
    const float NEG = -__builtin_huge_valf();
    float red = DOM == SBP_SUM ? 0.0f : NEG;
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        if (x < a.Ms) {
            hs[x] = h[q];
            red = DOM == SBP_SUM ? red + h[q] : fmaxf(red, h[q]);
        }
    }
    for (int off = 16; off; off >>= 1) {
        const float t = __shfl_xor_sync(SBP_FULL_MASK, red, off);
        red = DOM == SBP_SUM ? red + t : fmaxf(red, t);
    }
    __syncwarp();
    const float base = !a.floor_term ? (DOM == SBP_SUM ? 0.0f : NEG)
                                     : (DOM == SBP_SUM ? a.fbar[O] * red : a.fbar[O] + red);
    float out[ELL_QMAX];
    float tot = DOM == SBP_SUM ? 0.0f : NEG;
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        float acc = base;
        if (x < a.M) {
            const int *ip = a.idx[O] + x;
            const float *wp = a.w[O] + x;
            for (int k = 0; k < a.m_max; ++k) {
                const float hv = hs[ip[(long long)k * a.Ms]];
                const float w = wp[(long long)k * a.Ms];
                acc = DOM == SBP_SUM ? fmaf(w, hv, acc) : fmaxf(acc, w + hv);
            }
        } else {
            acc = DOM == SBP_SUM ? 0.0f : NEG;
        }
        out[q] = acc;
        if (x < a.Ms) tot = DOM == SBP_SUM ? tot + acc : fmaxf(tot, acc);
    }
    __syncwarp();
    for (int off = 16; off; off >>= 1) {
        const float t = __shfl_xor_sync(SBP_FULL_MASK, tot, off);
        tot = DOM == SBP_SUM ? tot + t : fmaxf(tot, t);
    }
    bool ok;
    if (DOM == SBP_SUM) {
        ok = (tot > 0.0f) && !isinf(tot);
        const float inv = __frcp_rn(tot);
#pragma unroll
        for (int q = 0; q < ELL_QMAX; ++q) out[q] *= inv;
    } else {
        ok = isfinite(tot);
#pragma unroll
        for (int q = 0; q < ELL_QMAX; ++q) out[q] -= tot;
    }
    if (!active) return;
    const long long W = a.W;
    const long long step = DIR == 0 ? 1 : DIR == 1 ? -1 : DIR == 2 ? W : -W;
    float *dst = a.msgs_out + dir_wslot(DIR) * a.slot_stride + (node_l + step) * a.Ms;
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        if (x < a.Ms) dst[x] = out[q];
    }
    if (!ok && lane == 0) report_failure(a.err, a.iteration, directed_edge_id(a.H, W, r, c, DIR));
}

template <int DOM>
__global__ void __launch_bounds__(32 * ELL_WARPS) ell_iter_kernel(const __grid_constant__ EllArgs a) {
    __shared__ float hs_all[ELL_WARPS][32 * ELL_QMAX];
    const int lane = threadIdx.x & 31;
    float *hs = hs_all[threadIdx.x >> 5];
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long p = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (p >= npix) return;   // warp-uniform
    const int lr = a.lr_begin + (int)(p / a.W);
    const int c = (int)(p % a.W);
    const long long r = (long long)a.r0 + lr - 1;
    const long long node_l = (long long)lr * a.W + c;
    const float *gp = a.values + ((long long)(lr - 1) * a.W + c) * a.Ms;
    const float *mp = a.msgs_in + node_l * a.Ms;
    const float PAD = DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    float g[ELL_QMAX], m[4][ELL_QMAX];
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        const bool in = x < a.Ms;
        g[q] = in ? gp[x] : PAD;
#pragma unroll
        if (!a.first) {
            for (int k = 0; k < 4; ++k) m[k][q] = in ? mp[k * a.slot_stride + x] : PAD;
        } else {
            const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
            for (int k = 0; k < 4; ++k)
                m[k][q] = x >= a.M ? PAD
                                   : (DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M) : 0.0f);
        }
    }
    float h[ELL_QMAX];
    const bool has_r = c + 1 < a.W, has_l = c > 0, has_d = r + 1 < a.H, has_u = r > 0;
    if (DOM == SBP_SUM) {
#define SBP_H(E0, E1, E2)                                                                  \
    for (int q = 0; q < ELL_QMAX; ++q) h[q] = ((g[q] * m[E0][q]) * m[E1][q]) * m[E2][q];
        if (has_u) { SBP_H(1, 2, 3) ell_emit<DOM, 3>(a, h, hs, lane, true, node_l, r, c); }
        if (has_l) { SBP_H(0, 2, 3) ell_emit<DOM, 1>(a, h, hs, lane, true, node_l, r, c); }
        if (has_r) { SBP_H(0, 1, 3) ell_emit<DOM, 0>(a, h, hs, lane, true, node_l, r, c); }
        if (has_d) { SBP_H(0, 1, 2) ell_emit<DOM, 2>(a, h, hs, lane, true, node_l, r, c); }
#undef SBP_H
    } else {
        // Same error-free (TwoSum) sums and shift as the band kernel, in the
        // same operation order, so fast (band) and standard (dense) max-sum
        // stay bit-identical as in the reference (bp.py:325-333).
        float sa[ELL_QMAX], ea[ELL_QMAX], s2[ELL_QMAX], e2[ELL_QMAX];
        for (int q = 0; q < ELL_QMAX; ++q) two_sum(g[q], m[0][q], sa[q], ea[q]);
        if (has_u) {
            for (int q = 0; q < ELL_QMAX; ++q) {
                float t, e;
                two_sum(g[q], m[1][q], s2[q], e2[q]);
                two_sum(s2[q], m[2][q], t, e); s2[q] = t; e2[q] += e;
                two_sum(s2[q], m[3][q], t, e); s2[q] = t; e2[q] += e;
            }
            shift_compensated<ELL_QMAX, 32>(s2, e2, h);
            ell_emit<DOM, 3>(a, h, hs, lane, true, node_l, r, c);
        }
        if (has_l) {
            for (int q = 0; q < ELL_QMAX; ++q) {
                float t, e;
                two_sum(sa[q], m[2][q], s2[q], e); e2[q] = ea[q] + e;
                two_sum(s2[q], m[3][q], t, e); s2[q] = t; e2[q] += e;
            }
            shift_compensated<ELL_QMAX, 32>(s2, e2, h);
            ell_emit<DOM, 1>(a, h, hs, lane, true, node_l, r, c);
        }
        for (int q = 0; q < ELL_QMAX; ++q) {
            float t, e;
            two_sum(sa[q], m[1][q], t, e); sa[q] = t; ea[q] += e;
        }
        if (has_r) {
            for (int q = 0; q < ELL_QMAX; ++q) {
                float e;
                two_sum(sa[q], m[3][q], s2[q], e); e2[q] = ea[q] + e;
            }
            shift_compensated<ELL_QMAX, 32>(s2, e2, h);
            ell_emit<DOM, 0>(a, h, hs, lane, true, node_l, r, c);
        }
        if (has_d) {
            for (int q = 0; q < ELL_QMAX; ++q) {
                float e;
                two_sum(sa[q], m[2][q], s2[q], e); e2[q] = ea[q] + e;
            }
            shift_compensated<ELL_QMAX, 32>(s2, e2, h);
            ell_emit<DOM, 2>(a, h, hs, lane, true, node_l, r, c);
        }
    }
}

cudaError_t launch_ell(int domain, const EllArgs &a, cudaStream_t s) {
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long blocks = (npix + ELL_WARPS - 1) / ELL_WARPS;
    if (blocks <= 0) return cudaSuccess;
    if (domain == SBP_SUM)
        ell_iter_kernel<SBP_SUM><<<(unsigned)blocks, 32 * ELL_WARPS, 0, s>>>(a);
    else
        ell_iter_kernel<SBP_MAX><<<(unsigned)blocks, 32 * ELL_WARPS, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace sbp
