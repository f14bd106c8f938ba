// General potentials: per-column compatible lists in ELL form, shared or
// per edge, for both schedules.
//
// Covers potentials that are not Toeplitz bands (arbitrary CSC, as produced
// by sparse_from_dense or the reference's random_sparse_potential,
// synth.py:21-43), per-edge (inhomogeneous) potentials -- which the reference
// runs on its generic engine in the same grid pass order (bp.py:506-584,
// 218-234) -- and, with m_max = M and idx[k][x] = k, the dense "standard"
// update (numba_kernels.py:35-41, 66-74) for small M.  One warp per node
// (synchronous) or per chain (sequential); h is staged in shared memory so
// the gather h[idx] is a broadcast / conflict-light LDS; the entries of a
// column are visited in ascending x_i, the reference order; padded entries
// carry weight 0 (sum) / -inf (max).
//
// Potential storage: `idx` / `w` point at [n_pot][2 orientations][m_max][Ms];
// with per-edge potentials pid_h[r*W + c] is the potential of edge
// (n, n+1) and pid_v[r*W + c] that of (n, n+W) (global node ids).  Messages
// from n to n+1 / n+W use orientation 0, to n-1 / n-W orientation 1 of the
// edge's potential (bp.py:525, 443-463).
#include "aux_kernels.cuh"
#include "band_kernel.cuh"   // two_sum, shift_compensated, lanes_max

namespace sbp {

constexpr int ELL_WARPS = 4;
constexpr int ELL_QMAX = 8;   // Ms <= 256

// Potential slot of the message node (r, c) -> direction dir.
__device__ __forceinline__ long long ell_pot_slot(const EllArgs &a, long long r, int c, int dir) {
    long long pid = 0;
    if (a.pid_h) {
        const long long n = r * a.W + c;
        pid = dir == 0 ? a.pid_h[n] : dir == 1 ? a.pid_h[n - 1]
            : dir == 2 ? a.pid_v[n] : a.pid_v[n - a.W];
    }
    return pid * 2 + dir_orient(dir);
}

// Exclusion vector h in the reference order (unary, slots 0..3 ascending,
// skipping excl); max-sum error-free with the node shift, as the band kernel.
template <int DOM>
__device__ __forceinline__ void ell_h(const float (&g)[ELL_QMAX], const float (&m)[4][ELL_QMAX],
                                      int excl, float (&h)[ELL_QMAX]) {
    if (DOM == SBP_SUM) {
#pragma unroll
        for (int q = 0; q < ELL_QMAX; ++q) {
            float v = g[q];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k != excl) v *= m[k][q];
            h[q] = v;
        }
    } else {
        float s[ELL_QMAX], e[ELL_QMAX];
#pragma unroll
        for (int q = 0; q < ELL_QMAX; ++q) {
            s[q] = g[q];
            e[q] = 0.0f;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k != excl) {
                    float t, ee;
                    two_sum(s[q], m[k][q], t, ee);
                    s[q] = t;
                    e[q] += ee;
                }
        }
        shift_compensated<ELL_QMAX, 32>(s, e, h);
    }
}

// Accurate sum-product (EllArgs::acc64): the exclusion products, S, the floor
// term, the correction and the normaliser in f64 (the reference's own
// precision, numba_kernels.py:44-54, 248-258) from the f32-stored inputs;
// weights carry f64 precision as a hi + lo pair of f32 planes, fbar as f64.
// Only the stored message is rounded to f32.  For weak smoothing with wide
// bands, where fp32 accumulation drifts past the 1e-5 parity bar.
__device__ __forceinline__ void ell_h64(const float (&g)[ELL_QMAX], const float (&m)[4][ELL_QMAX],
                                        int excl, double (&h)[ELL_QMAX]) {
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        double v = g[q];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k != excl) v *= (double)m[k][q];
        h[q] = v;
    }
}

__device__ __forceinline__ bool ell_message64(const EllArgs &a, const double (&h)[ELL_QMAX],
                                              double *hs, int lane, long long pslot,
                                              float (&out)[ELL_QMAX]) {
    double red = 0.0;
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        if (x < a.Ms) {
            hs[x] = h[q];
            red += h[q];
        }
    }
    for (int off = 16; off; off >>= 1) red += __shfl_xor_sync(SBP_FULL_MASK, red, off);
    __syncwarp();
    const double base = a.floor_term ? a.fbar64[pslot & 1] * red : 0.0;
    const long long off0 = pslot * a.pot_stride;
    double acc[ELL_QMAX];
    double tot = 0.0;
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        double v = base;
        if (x < a.M) {
            const int *ip = a.idx + off0 + x;
            const float *wp = a.w + off0 + x;
            const float *lp = a.w_lo + off0 + x;
            for (int k = 0; k < a.m_max; ++k) {
                const long long o = (long long)k * a.Ms;
                const double w = (double)wp[o] + (double)lp[o];
                v = fma(w, hs[ip[o]], v);
            }
        } else {
            v = 0.0;
        }
        acc[q] = v;
        if (x < a.Ms) tot += v;
    }
    __syncwarp();
    for (int off = 16; off; off >>= 1) tot += __shfl_xor_sync(SBP_FULL_MASK, tot, off);
    const double inv = 1.0 / tot;
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) out[q] = (float)(acc[q] * inv);
    return (tot > 0.0) && !isinf(tot);
}

// The message of one directed edge: floor term + ELL correction (or the dense
// sum when floor_term = 0 and the lists are full), then normalisation.
template <int DOM>
__device__ __forceinline__ bool ell_message(const EllArgs &a, const float (&h)[ELL_QMAX],
                                            float *hs, int lane, long long pslot,
                                            float (&out)[ELL_QMAX]) {
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
    const float fb = a.fbar_all ? a.fbar_all[pslot] : a.fbar[pslot & 1];
    const float base = !a.floor_term ? (DOM == SBP_SUM ? 0.0f : NEG)
                                     : (DOM == SBP_SUM ? fb * red : fb + red);
    const long long off0 = pslot * a.pot_stride;
    float tot = DOM == SBP_SUM ? 0.0f : NEG;
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        float acc = base;
        if (x < a.M) {
            const int *ip = a.idx + off0 + x;
            const float *wp = a.w + off0 + x;
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
    if (DOM == SBP_SUM) {
        const float inv = __frcp_rn(tot);
#pragma unroll
        for (int q = 0; q < ELL_QMAX; ++q) out[q] *= inv;
        return (tot > 0.0f) && !isinf(tot);
    }
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) out[q] -= tot;
    return isfinite(tot);
}

// max |out - old| over the lane's labels (old: the message being replaced;
// iteration 0 of a synchronous run: the reference initial message)
template <int DOM>
__device__ __forceinline__ float ell_delta(const EllArgs &a, const float *old, int lane,
                                          const float (&out)[ELL_QMAX], bool first) {
    float d = 0.0f;
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        if (x < a.M) {
            const float o = first ? (DOM == SBP_SUM ? 1.0f / (float)a.M : 0.0f) : old[x];
            d = fmaxf(d, fabsf(out[q] - o));
        }
    }
    return d;
}

__device__ __forceinline__ void ell_flush_delta(float *delta, float d) {
    for (int off = 16; off; off >>= 1) d = fmaxf(d, __shfl_xor_sync(SBP_FULL_MASK, d, off));
    if ((threadIdx.x & 31) == 0 && d > 0.0f) atomicMax(reinterpret_cast<int *>(delta), __float_as_int(d));
}

__device__ __forceinline__ void ell_store(const EllArgs &a, float *base, int lane,
                                          const float (&out)[ELL_QMAX]) {
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        if (x < a.Ms) base[x] = out[q];
    }
}

template <int DOM, int ACC>
__global__ void __launch_bounds__(32 * ELL_WARPS) ell_iter_kernel(const __grid_constant__ EllArgs a) {
    __shared__ double hs_all[ELL_WARPS][32 * ELL_QMAX];
    const int lane = threadIdx.x & 31;
    float *hs = reinterpret_cast<float *>(hs_all[threadIdx.x >> 5]);
    double *hs64 = hs_all[threadIdx.x >> 5];
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
    const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
    float g[ELL_QMAX], m[4][ELL_QMAX];
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        const bool in = x < a.Ms;
        g[q] = in ? gp[x] : PAD;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!a.first)
                m[k][q] = in ? mp[k * a.slot_stride + x] : PAD;
            else
                m[k][q] = x >= a.M ? PAD
                                   : (DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M) : 0.0f);
        }
    }
    const bool has[4] = {c + 1 < a.W, c > 0, r + 1 < a.H, r > 0};
    const long long W = a.W;
    float dmax = 0.0f;
#pragma unroll
    for (int dir = 0; dir < 4; ++dir) {
        if (!has[dir]) continue;
        float out[ELL_QMAX];
        bool ok;
        if constexpr (ACC && DOM == SBP_SUM) {
            double h[ELL_QMAX];
            ell_h64(g, m, dir_excl(dir), h);
            ok = ell_message64(a, h, hs64, lane, ell_pot_slot(a, r, c, dir), out);
        } else {
            float h[ELL_QMAX];
            ell_h<DOM>(g, m, dir_excl(dir), h);
            ok = ell_message<DOM>(a, h, hs, lane, ell_pot_slot(a, r, c, dir), out);
        }
        const long long step = dir == 0 ? 1 : dir == 1 ? -1 : dir == 2 ? W : -W;
        const long long off = dir_wslot(dir) * a.slot_stride + (node_l + step) * a.Ms;
        if (a.delta) dmax = fmaxf(dmax, ell_delta<DOM>(a, a.msgs_in + off, lane, out, a.first));
        ell_store(a, a.msgs_out + off, lane, out);
        if (!ok && lane == 0)
            report_failure(a.err, a.iteration, directed_edge_id(a.H, W, r, c, dir));
    }
    if (a.delta) ell_flush_delta(a.delta, dmax);
}

// Sequential (canonical) pass over chains, one warp per chain; see
// chain_kernel.cuh for the pass geometry and the failure key.
template <int DOM, int ACC>
__global__ void __launch_bounds__(32 * ELL_WARPS) ell_chain_kernel(const __grid_constant__ EllArgs a) {
    __shared__ double hs_all[ELL_WARPS][32 * ELL_QMAX];
    const int lane = threadIdx.x & 31;
    float *hs = reinterpret_cast<float *>(hs_all[threadIdx.x >> 5]);
    double *hs64 = hs_all[threadIdx.x >> 5];
    const int dir = a.pass;
    const long long H = a.H, W = a.W;
    const long long n_lines = dir <= 1 ? H : W, len = dir <= 1 ? W - 1 : H - 1;
    const long long stride = dir <= 1 ? W : 1;
    const long long step = dir == 0 ? 1 : dir == 1 ? -1 : dir == 2 ? W : -W;
    const long long origin = dir == 1 ? W - 1 : dir == 3 ? (H - 1) * W : 0;
    const int wslot = dir_wslot(dir), excl = dir_excl(dir);
    const long long line = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (line >= n_lines) return;   // warp-uniform
    const float PAD = DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    float *msgs = a.msgs_out;
    const long long S = a.slot_stride;
    long long src = line * stride + origin;
    float dmax = 0.0f;
    float chain[ELL_QMAX];
#pragma unroll
    for (int q = 0; q < ELL_QMAX; ++q) {
        const int x = lane + 32 * q;
        chain[q] = x < a.Ms ? msgs[wslot * S + (src + W) * a.Ms + x] : PAD;
    }
    for (long long pos = 0; pos < len; ++pos, src += step) {
        float g[ELL_QMAX], m[4][ELL_QMAX];
#pragma unroll
        for (int q = 0; q < ELL_QMAX; ++q) {
            const int x = lane + 32 * q;
            const bool in = x < a.Ms;
            g[q] = in ? a.values[src * a.Ms + x] : PAD;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                m[k][q] = k == wslot ? chain[q]
                        : (k == excl || !in) ? PAD : msgs[k * S + (src + W) * a.Ms + x];
        }
        const long long r = src / W;
        const int c = (int)(src % W);
        bool ok;
        if constexpr (ACC && DOM == SBP_SUM) {
            double h[ELL_QMAX];
            ell_h64(g, m, excl, h);
            ok = ell_message64(a, h, hs64, lane, ell_pot_slot(a, r, c, dir), chain);
        } else {
            float h[ELL_QMAX];
            ell_h<DOM>(g, m, excl, h);
            ok = ell_message<DOM>(a, h, hs, lane, ell_pot_slot(a, r, c, dir), chain);
        }
        if (a.delta)
            dmax = fmaxf(dmax, ell_delta<DOM>(a, msgs + wslot * S + (src + step + W) * a.Ms, lane,
                                              chain, false));
        ell_store(a, msgs + wslot * S + (src + step + W) * a.Ms, lane, chain);
        if (!ok && lane == 0) {
            const unsigned long long key = ((unsigned long long)a.iteration << 40) |
                                           ((unsigned long long)dir << 38) |
                                           (unsigned long long)(line * len + pos);
            atomicMin(a.err, key);
        }
        __syncwarp();
    }
    if (a.delta) ell_flush_delta(a.delta, dmax);
}

cudaError_t launch_ell(int domain, const EllArgs &a, cudaStream_t s) {
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long blocks = (npix + ELL_WARPS - 1) / ELL_WARPS;
    if (blocks <= 0) return cudaSuccess;
    if (domain == SBP_SUM && a.acc64)
        ell_iter_kernel<SBP_SUM, 1><<<(unsigned)blocks, 32 * ELL_WARPS, 0, s>>>(a);
    else if (domain == SBP_SUM)
        ell_iter_kernel<SBP_SUM, 0><<<(unsigned)blocks, 32 * ELL_WARPS, 0, s>>>(a);
    else
        ell_iter_kernel<SBP_MAX, 0><<<(unsigned)blocks, 32 * ELL_WARPS, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_ell_sweep(int domain, const EllArgs &a, cudaStream_t s) {
    for (int dir = 0; dir < 4; ++dir) {
        EllArgs b = a;
        b.pass = dir;
        const long long lines = dir <= 1 ? a.H : a.W;
        const long long len = dir <= 1 ? a.W - 1 : a.H - 1;
        if (len <= 0) continue;
        const long long blocks = (lines + ELL_WARPS - 1) / ELL_WARPS;
        if (domain == SBP_SUM && a.acc64)
            ell_chain_kernel<SBP_SUM, 1><<<(unsigned)blocks, 32 * ELL_WARPS, 0, s>>>(b);
        else if (domain == SBP_SUM)
            ell_chain_kernel<SBP_SUM, 0><<<(unsigned)blocks, 32 * ELL_WARPS, 0, s>>>(b);
        else
            ell_chain_kernel<SBP_MAX, 0><<<(unsigned)blocks, 32 * ELL_WARPS, 0, s>>>(b);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace sbp
