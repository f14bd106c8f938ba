// Dense O(M^2) comparison kernel: the reference "standard" update
// (numba_kernels.py:35-41 `_std_sum`, 66-74 `_std_max`) as a tiled SIMT
// product.  For one orientation the update of a set of (node, direction)
// rows is
//     sum: out[row][x_j] = sum_{x_i} f(x_i, x_j) h[row][x_i]      (a GEMM)
//     max: out[row][x_j] = max_{x_i} f(x_i, x_j) + h[row][x_i]    (a (max,+) product)
// A block owns a tile of DP = 32 nodes.  Phase 1: each warp reads a node's
// unary and four incoming vectors once and forms all four exclusion vectors h
// (same products / error-free max-sum sums as the band kernel, so fast and
// standard max-sum stay bit-identical) into shared memory, transposed
// [dir][x][node].  Phase 2: two passes, one per orientation (rows = the
// tile's right+down or left+up vectors, 64 rows), each multiplying with the
// oriented table streamed through shared memory in 32-row chunks (cp.async
// double buffer); register tiles of PT rows x 8 labels per thread.  Then each
// row is normalised (shuffle reductions across the label threads) and stored
// into the neighbour's slot.  Sum accumulates x_i in ascending order like the
// reference; max is exact.  The next tile's inputs are prefetched into L2
// while the current tile multiplies.
//
// Tensor cores are deliberately not used: BASELINE asks for the dense update
// as an FP32 SIMT comparison point, and the (max,+) product has no tensor-core
// form.
#include "aux_kernels.cuh"
#include "band_kernel.cuh"   // two_sum, fmax3, lanes_max / lanes_sum

namespace sbp {

constexpr int DP = 32;       // nodes per tile
constexpr int DROWS = 2 * DP;  // rows per orientation pass (two directions)
constexpr int DK = 32;       // table rows per pipeline stage
constexpr int DTHREADS = 256;

template <int MS>
struct DenseShape {
    static constexpr int TX = MS / 8;              // threads across labels (8 labels each)
    static constexpr int TY = DTHREADS / TX;       // threads across rows
    static constexpr int PT = DROWS / TY;          // rows per thread (within one direction)
    static constexpr int HT = DP + 4;              // h stored transposed [dir][x][node], padded
    static constexpr int Q = MS / 32;              // labels per lane in phase 1
    static_assert(PT >= 1 && TX <= 32 && DP % PT == 0, "unsupported Ms for the dense kernel");
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// Phase 1: warp-per-node formation of the four exclusion vectors.
template <int DOM, int MS>
__device__ __forceinline__ void dense_form_h(const DenseArgs &a, long long p0, long long npix,
                                             float *hs) {
    using S = DenseShape<MS>;
    constexpr int Q = S::Q;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const float PAD = DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf();
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
        float g[Q], m[4][Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int x = lane + 32 * q;
            g[q] = gp[x];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                m[k][q] = a.first ? (x >= a.M ? PAD
                                              : (DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M)
                                                                : 0.0f))
                                  : mp[k * a.slot_stride + x];
        }
        // dir d excludes slot dir_excl(d): 0 -> 2, 1 -> 1, 2 -> 3, 3 -> 0
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            float h[Q];
            if (DOM == SBP_SUM) {
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    float v = g[q];
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (k != dir_excl(d)) v *= m[k][q];
                    h[q] = v;
                }
            } else {
                // identical TwoSum sequence to band_kernel.cuh (prefix order)
                float sv[Q], ev[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    float s, e, t, ee;
                    if (d == 3) {
                        two_sum(g[q], m[1][q], s, e);
                        two_sum(s, m[2][q], t, ee); s = t; e += ee;
                        two_sum(s, m[3][q], t, ee); s = t; e += ee;
                    } else if (d == 1) {
                        float sa, ea;
                        two_sum(g[q], m[0][q], sa, ea);
                        two_sum(sa, m[2][q], s, ee); e = ea + ee;
                        two_sum(s, m[3][q], t, ee); s = t; e += ee;
                    } else {
                        float sa, ea;
                        two_sum(g[q], m[0][q], sa, ea);
                        two_sum(sa, m[1][q], t, ee); sa = t; ea += ee;
                        two_sum(sa, d == 0 ? m[3][q] : m[2][q], s, ee); e = ea + ee;
                    }
                    sv[q] = s;
                    ev[q] = e;
                }
                shift_compensated<Q, 32>(sv, ev, h);
            }
#pragma unroll
            for (int q = 0; q < Q; ++q) hs[(d * MS + lane + 32 * q) * S::HT + pl] = h[q];
        }
    }
}

__device__ __forceinline__ void dense_prefetch_tile(const DenseArgs &a, long long p0,
                                                    long long npix) {
    const int lane = threadIdx.x;
    if (lane > 4 || p0 >= npix || (lane < 4 && a.first)) return;
    const long long n = npix - p0 < DP ? npix - p0 : DP;
    const unsigned bytes = (unsigned)(n * a.Ms * 4);
    const float *src = lane == 4
        ? a.values + ((long long)(a.lr_begin - 1) * a.W + p0) * a.Ms
        : a.msgs_in + lane * a.slot_stride + ((long long)a.lr_begin * a.W + p0) * a.Ms;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

template <int DOM, int MS>
__global__ void __launch_bounds__(DTHREADS, 1) dense_iter_kernel(const __grid_constant__ DenseArgs a) {
    using S = DenseShape<MS>;
    extern __shared__ __align__(16) float smem[];
    float *hs = smem;                               // [4][MS][HT]
    float *ts = smem + 4 * MS * S::HT;              // [2][DK][MS] (HT*4 B rows keep 16 B alignment)
    const int tid = threadIdx.x;
    const int tx = tid % S::TX, ty = tid / S::TX;
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long tiles = (npix + DP - 1) / DP;
    const float NEG = -__builtin_huge_valf();
    const long long W = a.W;

    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const long long p0 = tile * DP;
        __syncthreads();   // the previous tile is done with hs
        dense_form_h<DOM, MS>(a, p0, npix, hs);
        dense_prefetch_tile(a, p0 + (long long)gridDim.x * DP, npix);
#pragma unroll 1
        for (int o = 0; o < 2; ++o) {
            const float *tab = a.t[o];   // [MS][MS], f(x_i = k, x_j = x)
            auto load_stage = [&](int stage, int k0) {
                float *dst = ts + stage * DK * MS;
                for (int v = tid; v < DK * MS / 4; v += DTHREADS) {
                    const int row = v / (MS / 4), col4 = v % (MS / 4);
                    cp_async16(dst + row * MS + col4 * 4,
                               tab + (long long)(k0 + row) * MS + col4 * 4);
                }
                cp_async_commit();
            };
            // this thread's rows: direction dr (o = 0: right/down, 1: left/up), nodes pl0..
            const int row0 = ty * S::PT;
            const int dr = o == 0 ? (row0 < DP ? 0 : 2) : (row0 < DP ? 1 : 3);
            const int pl0 = row0 % DP;
            float acc[S::PT][8];
#pragma unroll
            for (int i = 0; i < S::PT; ++i)
#pragma unroll
                for (int l = 0; l < 8; ++l) acc[i][l] = DOM == SBP_SUM ? 0.0f : NEG;
            constexpr int NCH = MS / DK;
            __syncthreads();   // hs complete; ts free
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
                const float *hcol = hs + ((long long)dr * MS + ch * DK) * S::HT + pl0;
                // sum: one FFMA per term, x_i ascending; max: two terms per FMNMX3
                constexpr int KS = DOM == SBP_SUM ? 1 : 2;
#pragma unroll 4
                for (int kk = 0; kk < DK; kk += KS) {
                    float bv[KS][8], hv[KS][S::PT];
#pragma unroll
                    for (int u = 0; u < KS; ++u) {
                        const float4 b0 =
                            *reinterpret_cast<const float4 *>(tsc + (kk + u) * MS + tx * 4);
                        const float4 b1 = *reinterpret_cast<const float4 *>(
                            tsc + (kk + u) * MS + MS / 2 + tx * 4);
                        bv[u][0] = b0.x; bv[u][1] = b0.y; bv[u][2] = b0.z; bv[u][3] = b0.w;
                        bv[u][4] = b1.x; bv[u][5] = b1.y; bv[u][6] = b1.z; bv[u][7] = b1.w;
                        const float *hrow = hcol + (kk + u) * S::HT;
                        if constexpr (S::PT % 4 == 0) {
#pragma unroll
                            for (int i = 0; i < S::PT; i += 4) {
                                const float4 v = *reinterpret_cast<const float4 *>(hrow + i);
                                hv[u][i] = v.x; hv[u][i + 1] = v.y;
                                hv[u][i + 2] = v.z; hv[u][i + 3] = v.w;
                            }
                        } else {
#pragma unroll
                            for (int i = 0; i < S::PT; ++i) hv[u][i] = hrow[i];
                        }
                    }
                    // label pairs in packed FP32 (FFMA2 / FADD2): same roundings
#pragma unroll
                    for (int i = 0; i < S::PT; ++i)
#pragma unroll
                        for (int l = 0; l < 8; l += 2) {
                            if (DOM == SBP_SUM) {
                                fma2(acc[i][l], acc[i][l + 1], make_float2(bv[0][l], bv[0][l + 1]),
                                     hv[0][i]);
                            } else {
                                float a0, a1, b0, b1;
                                add2(a0, a1, bv[0][l], bv[0][l + 1], hv[0][i], hv[0][i]);
                                add2(b0, b1, bv[KS - 1][l], bv[KS - 1][l + 1], hv[KS - 1][i],
                                     hv[KS - 1][i]);
                                acc[i][l] = fmax3(acc[i][l], a0, b0);
                                acc[i][l + 1] = fmax3(acc[i][l + 1], a1, b1);
                            }
                        }
                }
                __syncthreads();
            }
            // normalise each row across the TX label threads, then store
#pragma unroll
            for (int i = 0; i < S::PT; ++i) {
                long long p = p0 + pl0 + i;
                const bool valid = p < npix;
                if (!valid) p = npix - 1;
                const int lr = a.lr_begin + (int)(p / a.W);
                const int c = (int)(p % a.W);
                const long long r = (long long)a.r0 + lr - 1;
                const bool exists = dr == 0 ? c + 1 < a.W : dr == 1 ? c > 0
                                  : dr == 2 ? r + 1 < a.H : r > 0;
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
                const long long step = dr == 0 ? 1 : dr == 1 ? -1 : dr == 2 ? W : -W;
                float *dst = a.msgs_out + dir_wslot(dr) * a.slot_stride + (node_l + step) * a.Ms;
                *reinterpret_cast<float4 *>(dst + tx * 4) =
                    make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
                *reinterpret_cast<float4 *>(dst + MS / 2 + tx * 4) =
                    make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
                if (!ok && tx == 0)
                    report_failure(a.err, a.iteration, directed_edge_id(a.H, W, r, c, dr));
            }
        }
    }
}

template <int DOM, int MS>
static cudaError_t launch_dense_ms(const DenseArgs &a, cudaStream_t s) {
    using S = DenseShape<MS>;
    const size_t smem = (4 * MS * S::HT + 2 * DK * MS) * sizeof(float);
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
