// Dense O(M^2) comparison kernel: the reference "standard" update
// (numba_kernels.py:35-41 `_std_sum`, 66-74 `_std_max`) as a tiled SIMT
// product.  For one orientation the update of P nodes is
//     sum: out[p][x_j] = sum_{x_i} f(x_i, x_j) h[p][x_i]      (a GEMM)
//     max: out[p][x_j] = max_{x_i} f(x_i, x_j) + h[p][x_i]    (a (max,+) product)
// A block owns P = 64 nodes and the full label row (Ms <= 256).  Per outgoing
// direction: warps form h for the tile (the same products / error-free
// max-sum sums as the band kernel, so fast and standard max-sum agree bit for
// bit) into shared memory, the block multiplies it with the oriented table
// streamed through shared memory in 32-row chunks (cp.async double buffer),
// then normalises each node's row (shuffle reductions across the label
// threads) and stores it into the neighbour's slot.  Sum accumulates x_i in
// ascending order like the reference; max is exact.
//
// Tensor cores are deliberately not used: BASELINE asks for the dense update
// as an FP32 SIMT comparison point, and the (max,+) product has no tensor-core
// form.
#include "aux_kernels.cuh"
#include "band_kernel.cuh"   // two_sum, lanes_max / lanes_sum

namespace sbp {

constexpr int DP = 64;       // nodes per block
constexpr int DK = 32;       // table rows per pipeline stage
constexpr int DTHREADS = 256;

template <int MS>
struct DenseShape {
    static constexpr int TX = MS / 8;              // threads across labels (8 labels each)
    static constexpr int TY = DTHREADS / TX;       // threads across nodes
    static constexpr int PT = DP / TY;             // nodes per thread
    static constexpr int HS = MS + 1;              // padded h row stride (floats)
    static_assert(PT >= 1 && TX <= 32, "unsupported Ms for the dense kernel");
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Warp-per-node h formation for one direction; writes h[p][x] (x < MS).
template <int DOM, int MS, int DIR>
__device__ __forceinline__ void dense_form_h(const DenseArgs &a, long long p0, long long npix,
                                             float *hs) {
    constexpr int Q = MS / 32 > 0 ? MS / 32 : 1;
    constexpr int HS = DenseShape<MS>::HS;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const float PAD = DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    constexpr int EXCL = dir_excl(DIR);
    for (int pl = warp; pl < DP; pl += DTHREADS / 32) {
        long long p = p0 + pl;
        if (p >= npix) p = npix - 1;
        const int lr = a.lr_begin + (int)(p / a.W);
        const int c = (int)(p % a.W);
        const long long r = (long long)a.r0 + lr - 1;
        const long long node_l = (long long)lr * a.W + c;
        const float *gp = a.values + ((long long)(lr - 1) * a.W + c) * a.Ms;
        const float *mp = a.msgs_in + node_l * a.Ms;
        const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
        float h[Q];
        float sv[Q], ev[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int x = lane + 32 * q;
            const bool in = x < MS;
            float m[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (a.first)
                    m[k] = x >= a.M ? PAD
                                    : (DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M) : 0.0f);
                else
                    m[k] = in ? mp[k * a.slot_stride + x] : PAD;
            }
            const float g = in ? gp[x] : PAD;
            if (DOM == SBP_SUM) {
                float v = g;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (k != EXCL) v *= m[k];
                h[q] = v;
            } else {
                // identical TwoSum sequence to band_kernel.cuh (prefix order)
                float s, e;
                if (EXCL == 0) {
                    float t, ee;
                    two_sum(g, m[1], s, e);
                    two_sum(s, m[2], t, ee); s = t; e += ee;
                    two_sum(s, m[3], t, ee); s = t; e += ee;
                } else if (EXCL == 1) {
                    float sa, ea, t, ee;
                    two_sum(g, m[0], sa, ea);
                    two_sum(sa, m[2], s, ee); e = ea + ee;
                    two_sum(s, m[3], t, ee); s = t; e += ee;
                } else {
                    float sa, ea, t, ee;
                    two_sum(g, m[0], sa, ea);
                    two_sum(sa, m[1], t, ee); sa = t; ea += ee;
                    two_sum(sa, EXCL == 2 ? m[3] : m[2], s, ee); e = ea + ee;
                }
                sv[q] = s;
                ev[q] = e;
            }
        }
        if (DOM == SBP_MAX) {
            float cmax = sv[0];
#pragma unroll
            for (int q = 1; q < Q; ++q) cmax = fmaxf(cmax, sv[q]);
            cmax = lanes_max<32>(cmax);
            if (!isfinite(cmax)) cmax = 0.0f;
#pragma unroll
            for (int q = 0; q < Q; ++q) h[q] = (sv[q] - cmax) + ev[q];
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int x = lane + 32 * q;
            if (x < MS) hs[pl * HS + x] = h[q];
        }
    }
}

template <int DOM, int MS>
__global__ void __launch_bounds__(DTHREADS, 1) dense_iter_kernel(const __grid_constant__ DenseArgs a) {
    using S = DenseShape<MS>;
    extern __shared__ __align__(16) float smem[];
    float *hs = smem;                               // [DP][HS]
    float *ts = smem + DP * S::HS + 3;              // [2][DK][MS], 16-byte aligned below
    ts = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(ts) + 15) & ~uintptr_t(15));
    const int tid = threadIdx.x;
    const int tx = tid % S::TX, ty = tid / S::TX;
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long tiles = (npix + DP - 1) / DP;
    const float NEG = -__builtin_huge_valf();

    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const long long p0 = tile * DP;
#pragma unroll 1
        for (int dir = 0; dir < 4; ++dir) {
            __syncthreads();   // previous direction finished with hs / ts
            switch (dir) {
            case 0: dense_form_h<DOM, MS, 0>(a, p0, npix, hs); break;
            case 1: dense_form_h<DOM, MS, 1>(a, p0, npix, hs); break;
            case 2: dense_form_h<DOM, MS, 2>(a, p0, npix, hs); break;
            default: dense_form_h<DOM, MS, 3>(a, p0, npix, hs); break;
            }
            const float *tab = a.t[dir_orient(dir)];   // [MS][MS], f(x_i = k, x_j = x)
            auto load_stage = [&](int stage, int k0) {
                float *dst = ts + stage * DK * MS;
                for (int v = tid; v < DK * MS / 4; v += DTHREADS) {
                    const int row = v / (MS / 4), col4 = v % (MS / 4);
                    cp_async16(dst + row * MS + col4 * 4, tab + (long long)(k0 + row) * MS + col4 * 4);
                }
                cp_async_commit();
            };
            float acc[S::PT][8];
#pragma unroll
            for (int i = 0; i < S::PT; ++i)
#pragma unroll
                for (int l = 0; l < 8; ++l) acc[i][l] = DOM == SBP_SUM ? 0.0f : NEG;
            constexpr int NCH = (MS + DK - 1) / DK;
            load_stage(0, 0);
            for (int ch = 0; ch < NCH; ++ch) {
                if (ch + 1 < NCH) {
                    load_stage((ch + 1) & 1, (ch + 1) * DK);
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();
                const float *tsc = ts + (ch & 1) * DK * MS;
                const int kmax = MS - ch * DK < DK ? MS - ch * DK : DK;
#pragma unroll 4
                for (int kk = 0; kk < kmax; ++kk) {
                    const int k = ch * DK + kk;
                    const float4 b0 = *reinterpret_cast<const float4 *>(tsc + kk * MS + tx * 4);
                    const float4 b1 =
                        *reinterpret_cast<const float4 *>(tsc + kk * MS + MS / 2 + tx * 4);
                    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                    for (int i = 0; i < S::PT; ++i) {
                        const float hv = hs[(ty * S::PT + i) * S::HS + k];
#pragma unroll
                        for (int l = 0; l < 8; ++l) {
                            if (DOM == SBP_SUM) acc[i][l] = fmaf(bv[l], hv, acc[i][l]);
                            else acc[i][l] = fmaxf(acc[i][l], bv[l] + hv);
                        }
                    }
                }
                __syncthreads();
            }
            // normalise each node row across the TX label threads, then store
            const long long W = a.W;
#pragma unroll
            for (int i = 0; i < S::PT; ++i) {
                long long p = p0 + ty * S::PT + i;
                const bool valid = p < npix;
                if (!valid) p = npix - 1;
                const int lr = a.lr_begin + (int)(p / a.W);
                const int c = (int)(p % a.W);
                const long long r = (long long)a.r0 + lr - 1;
                const bool exists = dir == 0 ? c + 1 < a.W : dir == 1 ? c > 0
                                  : dir == 2 ? r + 1 < a.H : r > 0;
                float red = DOM == SBP_SUM ? 0.0f : NEG;
#pragma unroll
                for (int l = 0; l < 8; ++l) {
                    const int x = l < 4 ? tx * 4 + l : MS / 2 + tx * 4 + (l - 4);
                    if (x >= a.M) acc[i][l] = DOM == SBP_SUM ? 0.0f : NEG;
                    red = DOM == SBP_SUM ? red + acc[i][l] : fmaxf(red, acc[i][l]);
                }
                red = DOM == SBP_SUM ? lanes_sum<S::TX>(red) : lanes_max<S::TX>(red);
                bool ok;
                if (DOM == SBP_SUM) {
                    ok = (red > 0.0f) && !isinf(red);
                    const float inv = __frcp_rn(red);
#pragma unroll
                    for (int l = 0; l < 8; ++l) acc[i][l] *= inv;
                } else {
                    ok = isfinite(red);
#pragma unroll
                    for (int l = 0; l < 8; ++l) acc[i][l] -= red;
                }
                if (!(valid && exists)) continue;
                const long long node_l = (long long)lr * W + c;
                const long long step = dir == 0 ? 1 : dir == 1 ? -1 : dir == 2 ? W : -W;
                float *dst = a.msgs_out + dir_wslot(dir) * a.slot_stride + (node_l + step) * a.Ms;
                *reinterpret_cast<float4 *>(dst + tx * 4) =
                    make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                *reinterpret_cast<float4 *>(dst + MS / 2 + tx * 4) =
                    make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
                if (!ok && tx == 0)
                    report_failure(a.err, a.iteration, directed_edge_id(a.H, W, r, c, dir));
            }
        }
    }
}

template <int DOM, int MS>
static cudaError_t launch_dense_ms(const DenseArgs &a, cudaStream_t s) {
    using S = DenseShape<MS>;
    const size_t smem = (DP * S::HS + 8) * sizeof(float) + 2 * DK * MS * sizeof(float);
    static bool configured = false;
    static int sms = 0;
    if (!configured) {
        cudaFuncSetAttribute(dense_iter_kernel<DOM, MS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        configured = true;
    }
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    long long tiles = (npix + DP - 1) / DP;
    if (tiles <= 0) return cudaSuccess;
    if (tiles > sms) tiles = sms;
    dense_iter_kernel<DOM, MS><<<(unsigned)tiles, DTHREADS, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_dense(int domain, const DenseArgs &a, cudaStream_t s) {
#define SBP_D(MSV)                                                                  \
    case MSV:                                                                       \
        return domain == SBP_SUM ? launch_dense_ms<SBP_SUM, MSV>(a, s)              \
                                 : launch_dense_ms<SBP_MAX, MSV>(a, s);
    switch (a.Ms) {
        SBP_D(32) SBP_D(64) SBP_D(128) SBP_D(256)
    default: return cudaErrorNotSupported;
    }
#undef SBP_D
}

}  // namespace sbp
