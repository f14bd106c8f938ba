// Dense O(M^2) sum-product update on the 5th-generation tensor cores (sm_100a
// tcgen05 + tensor memory): the reference "standard" update
// (numba_kernels.py:35-41 `_std_sum`, _grid_h_sum :194-210, _norm_sum_store
// :248-259) of one synchronous iteration as the GEMM it is,
//
//     out[x_i][n] = sum_{x_j} f(x_i, x_j) h[x_j][n],   n = (node, direction),
//
// in 3xTF32: f = f_hi + f_lo, h = h_hi + h_lo (hi = the value rounded to
// tf32, lo = the exact fp32 remainder), out = f_hi h_lo + f_lo h_hi + f_hi h_hi
// accumulated in fp32 by the tensor core (the dropped f_lo h_lo term is
// 2^-22 relative).  Symmetric tables only (one resident copy serves both
// orientations), Ms = 128 (one CTA) or Ms = 256 (a CTA pair, cta_group::2,
// each CTA owning 128 of the 256 output labels).
//
// Layout per CTA:
//   shared memory  f_hi rows of this CTA [128 x Ms] tf32, K-major, 128-byte swizzle (64 / 128 KB)
//                  3 stages of the h tile: [32 / CG columns x Ms] hi and lo planes (32 KB each)
//   tensor memory  columns [0, 96): 3 accumulator stages [128 labels x 32 columns] fp32
//                  columns [128, 128 + Ms): f_lo rows of this CTA (the A operand of f_lo h_hi)
// Warp roles (17 warps, one CTA per SM, persistent over tiles of 8 nodes):
//   warps 0-3    epilogue: tcgen05.ld the accumulator (thread = output label),
//                scale by the column's 1/s, store into the neighbour's slot
//                (a warp stores 128 contiguous bytes per column)
//   warp 4       allocates tensor memory; one elected thread of the leader CTA
//                issues the 3 Ms/8 tcgen05.mma of a tile and commits to an mbarrier
//   warps 5-16   producers, 3 groups of 4 warps, group g fills stage g: read the
//                unary and the four incoming messages of the tile's nodes once,
//                form the four exclusion products in the reference order, split
//                hi / lo straight into the swizzled operand rows, and compute the
//                normaliser s = sum_{x_j} colsum_f(x_j) h(x_j) (equal to the sum of
//                the outputs up to rounding; the reference divides by that sum)
// mbarriers per stage: full (producers -> MMA), accf (MMA commit -> epilogue),
// invf (producers -> epilogue: the 1/s values), free (epilogue -> producers).
#include "aux_kernels.cuh"
#include "band_kernel.cuh"   // vmul, lanes_sum, smem_u32, mbar_init

namespace sbp {
namespace tc {

constexpr int TC_NODES = 8;                 // nodes per tile
constexpr int TC_N = 4 * TC_NODES;          // MMA N: (node, direction) columns per tile
constexpr int TC_STAGES = 3;
constexpr int TC_EPI_WARPS = 4;
constexpr int TC_PROD_WARPS = 4 * TC_STAGES;
constexpr int TC_WARPS = TC_EPI_WARPS + 1 + TC_PROD_WARPS;
constexpr int TC_THREADS = 32 * TC_WARPS;   // 544
constexpr int TC_ACOL = 128;                // tensor-memory column of f_lo

template <int MS>
struct TcShape {
    static constexpr int CG = MS / 128;               // CTAs per MMA (cta_group)
    static constexpr int NB = TC_N / CG;              // h-tile columns held by one CTA
    static constexpr int KA = MS / 32;                // 128-byte swizzle atoms along K
    static constexpr int A_ATOM = 128 * 128;          // bytes: 128 rows x 32 tf32
    static constexpr int B_ATOM = NB * 128;
    static constexpr int A_BYTES = KA * A_ATOM;
    static constexpr int B_PLANE = KA * B_ATOM;
    static constexpr int STAGE_BYTES = 2 * B_PLANE;   // hi and lo planes
    static constexpr int LP = MS / 8;                 // lanes per node (8 labels each)
    static constexpr int NPW = 32 / LP;               // nodes per producer warp
    static constexpr int NCTA = TC_NODES / CG;        // nodes of a tile formed by one CTA
    static constexpr int TCOLS = MS == 128 ? 256 : 512;
    static constexpr int AUX_BYTES = 2048;            // colsum, 1/s, mbarriers, tmem address
    static constexpr size_t SMEM = (size_t)A_BYTES + TC_STAGES * STAGE_BYTES + AUX_BYTES;
    static_assert(MS == 128 || MS == 256, "tensor-core dense kernel: Ms = 128 or 256");
    static_assert(NPW * 4 == NCTA, "four producer warps form one CTA's share of a tile");
};

// ---- PTX helpers -----------------------------------------------------------

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// shared::cta address -> shared::cluster address of the same offset in CTA `rank`
__device__ __forceinline__ unsigned mapa(unsigned addr, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}

template <int CG>
__device__ __forceinline__ void bar_arrive(unsigned long long *bar, unsigned rank) {
    if (CG == 1)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
    else
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                         mapa(smem_u32(bar), rank)) : "memory");
}

// Bounded spin: a protocol error traps instead of hanging the device.
template <int CG>
__device__ __forceinline__ void bar_wait(unsigned long long *bar, unsigned parity) {
    unsigned done = 0;
    for (unsigned spin = 0; !done; ++spin) {
        if (CG == 1)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
                         " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        else
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                         " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (spin > (1u << 27)) __trap();
    }
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ float tf32_rna(float x) {
    unsigned u;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
    return __uint_as_float(u);
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm_100 descriptor
// version 1): rows of 128 bytes (32 tf32), 8-row groups 1024 bytes apart
// (stride byte offset), the 16-byte chunk c of row r stored at chunk c ^ (r % 8);
// validated on B200 by tools/tc_probe.cu.
__device__ __forceinline__ unsigned long long sw128_desc(unsigned saddr) {
    return (unsigned long long)((saddr & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}

// byte offset of the 16-byte chunk `ch` (4 consecutive k) of row `row`
__device__ __forceinline__ int sw128_chunk(int row, int ch, int atom_bytes) {
    return (ch >> 3) * atom_bytes + (row >> 3) * 1024 + (row & 7) * 128 + (((ch & 7) ^ (row & 7)) << 4);
}

template <int CG>
__device__ __forceinline__ void mma_ss(unsigned d, unsigned long long a, unsigned long long b, unsigned idesc,
                                       unsigned acc) {
    if (CG == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b),
                     "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b),
                     "r"(idesc), "r"(acc) : "memory");
}

template <int CG>
__device__ __forceinline__ void mma_ts(unsigned d, unsigned a_tmem, unsigned long long b, unsigned idesc,
                                       unsigned acc) {
    if (CG == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem),
                     "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem),
                     "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int CG>
__device__ __forceinline__ void mma_commit(unsigned long long *bar) {
    if (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(bar)) : "memory");
    else
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
                     "[%0], %1;" ::"r"(smem_u32(bar)), "h"((unsigned short)3) : "memory");
}

__device__ __forceinline__ void tmem_ld32(unsigned taddr, float (&v)[32]) {
    unsigned r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,"
        "%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st32(unsigned taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,"
        "%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
        "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
        "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
        "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
        "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
        "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
        : "memory");
}

__device__ __forceinline__ void sts128(unsigned saddr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__device__ __forceinline__ void l2_prefetch(const void *p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- the kernel --------------------------------------------------------------

template <int MS>
__global__ void __launch_bounds__(TC_THREADS, 1) dense_tc_kernel(const __grid_constant__ DenseArgs a) {
    using S = TcShape<MS>;
    constexpr int CG = S::CG;
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    unsigned char *sA = tc_smem;
    unsigned char *sB = tc_smem + S::A_BYTES;
    float *csum = reinterpret_cast<float *>(sB + TC_STAGES * S::STAGE_BYTES);   // [MS]
    float *inv = csum + MS;                                                     // [stage][32]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(inv + TC_STAGES * TC_N);
    unsigned long long *full = bars, *accf = bars + TC_STAGES, *invf = bars + 2 * TC_STAGES,
                       *freeb = bars + 3 * TC_STAGES;
    unsigned *tmem_slot = reinterpret_cast<unsigned *>(bars + 4 * TC_STAGES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned rank = CG == 2 ? cluster_rank() : 0u;
    const long long cluster = blockIdx.x / CG, nclusters = gridDim.x / CG;
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long tiles = (npix + TC_NODES - 1) / TC_NODES;
    const float *tab = a.t[0];

    // ---- one-time setup: f_hi -> shared memory, column sums, barriers, tensor memory
    for (int i = tid; i < 128 * (MS / 4); i += TC_THREADS) {
        const int row = i / (MS / 4), ch = i % (MS / 4);
        const float4 v = *reinterpret_cast<const float4 *>(tab + (size_t)(128 * rank + row) * MS + 4 * ch);
        sts128(smem_u32(sA) + sw128_chunk(row, ch, S::A_ATOM), tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z),
               tf32_rna(v.w));
    }
    {
        // column sums of the whole table, fixed order: SL row slices, then the slices
        constexpr int SL = 2;
        float *part = reinterpret_cast<float *>(sB);   // [SL][MS] scratch in stage 0
        if (tid < SL * MS) {
            const int x = tid % MS, sl = tid / MS;
            float s = 0.0f;
#pragma unroll 16
            for (int k = sl * (MS / SL); k < (sl + 1) * (MS / SL); ++k) s += tab[(size_t)k * MS + x];
            part[sl * MS + x] = s;
        }
        __syncthreads();
        if (tid < MS) {
            float s = 0.0f;
            for (int sl = 0; sl < SL; ++sl) s += part[sl * MS + tid];
            csum[tid] = s;
        }
    }
    if (tid == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(&full[s], 4 * CG);
            mbar_init(&accf[s], 1);
            mbar_init(&invf[s], 4 * CG);
            mbar_init(&freeb[s], TC_EPI_WARPS * CG);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == TC_EPI_WARPS) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)), "n"(S::TCOLS) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)), "n"(S::TCOLS) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem = *tmem_slot;
    if (warp < TC_EPI_WARPS) {
        // f_lo rows of this CTA -> tensor memory: lane = label row, column = k
        const float *row = tab + (size_t)(128 * rank + 32 * warp + lane) * MS;
        for (int k0 = 0; k0 < MS; k0 += 32) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                const float4 t = *reinterpret_cast<const float4 *>(row + k0 + i);
                v[i] = t.x - tf32_rna(t.x);
                v[i + 1] = t.y - tf32_rna(t.y);
                v[i + 2] = t.z - tf32_rna(t.z);
                v[i + 3] = t.w - tf32_rna(t.w);
            }
            tmem_st32(tmem + ((unsigned)(32 * warp) << 16) + TC_ACOL + k0, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async;" ::: "memory");   // f_hi: generic-proxy writes -> tensor-core reads
    tc_fence_before();
    __syncthreads();
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    tc_fence_after();

    if (warp < TC_EPI_WARPS) {
        // ================= epilogue =================
        const int x = 128 * (int)rank + 32 * warp + lane;   // output label of this thread
        const long long W = a.W;
        long long i = 0;
        for (long long tile = cluster; tile < tiles; tile += nclusters, ++i) {
            const int s = (int)(i % TC_STAGES);
            const unsigned par = (unsigned)((i / TC_STAGES) & 1);
            bar_wait<CG>(&invf[s], par);
            bar_wait<CG>(&accf[s], par);
            tc_fence_after();
            float v[32];
            tmem_ld32(tmem + ((unsigned)(32 * warp) << 16) + TC_N * s, v);
            const float *iv = inv + s * TC_N;
            const long long p0 = tile * TC_NODES;
            int lr = a.lr_begin + (int)(p0 / W);
            int c = (int)(p0 % W);
#pragma unroll
            for (int n = 0; n < TC_NODES; ++n) {
                if (p0 + n < npix) {
                    const long long r = (long long)a.r0 + lr - 1;
                    const long long node_l = (long long)lr * W + c;
                    float *base = a.msgs_out + node_l * a.Ms + x;
                    if (c + 1 < a.W) base[dir_wslot(0) * a.slot_stride + a.Ms] = v[4 * n + 0] * iv[4 * n + 0];
                    if (c > 0) base[dir_wslot(1) * a.slot_stride - a.Ms] = v[4 * n + 1] * iv[4 * n + 1];
                    if (r + 1 < a.H) base[dir_wslot(2) * a.slot_stride + W * a.Ms] = v[4 * n + 2] * iv[4 * n + 2];
                    if (r > 0) base[dir_wslot(3) * a.slot_stride - W * a.Ms] = v[4 * n + 3] * iv[4 * n + 3];
                }
                if (++c == a.W) { c = 0; ++lr; }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                bar_arrive<CG>(&freeb[s], rank);
                if (CG == 2) bar_arrive<CG>(&freeb[s], rank ^ 1u);
            }
        }
    } else if (warp == TC_EPI_WARPS) {
        // ================= MMA issuer (leader CTA) =================
        if (rank == 0) {
            const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(TC_N >> 3) << 17) |
                                   ((unsigned)((128 * CG) >> 4) << 24);
            const unsigned sA_u = smem_u32(sA), sB_u = smem_u32(sB);
            long long i = 0;
            for (long long tile = cluster; tile < tiles; tile += nclusters, ++i) {
                const int s = (int)(i % TC_STAGES);
                const unsigned par = (unsigned)((i / TC_STAGES) & 1);
                bar_wait<CG>(&full[s], par);
                tc_fence_after();
                if (lane == 0) {
                    const unsigned d = tmem + TC_N * s;
                    const unsigned bhi = sB_u + s * S::STAGE_BYTES, blo = bhi + S::B_PLANE;
                    // f_hi h_lo, f_lo h_hi (small terms first), then f_hi h_hi
#pragma unroll 4
                    for (int k = 0; k < MS / 8; ++k)
                        mma_ss<CG>(d, sw128_desc(sA_u + (k >> 2) * S::A_ATOM + (k & 3) * 32),
                                   sw128_desc(blo + (k >> 2) * S::B_ATOM + (k & 3) * 32), idesc, k > 0);
#pragma unroll 4
                    for (int k = 0; k < MS / 8; ++k)
                        mma_ts<CG>(d, tmem + TC_ACOL + 8 * k,
                                   sw128_desc(bhi + (k >> 2) * S::B_ATOM + (k & 3) * 32), idesc, 1u);
#pragma unroll 4
                    for (int k = 0; k < MS / 8; ++k)
                        mma_ss<CG>(d, sw128_desc(sA_u + (k >> 2) * S::A_ATOM + (k & 3) * 32),
                                   sw128_desc(bhi + (k >> 2) * S::B_ATOM + (k & 3) * 32), idesc, 1u);
                    mma_commit<CG>(&accf[s]);
                }
                __syncwarp();
            }
        }
    } else {
        // ================= producers =================
        constexpr int LP = S::LP, NPW = S::NPW;
        const int pw = warp - TC_EPI_WARPS - 1;
        const int grp = pw / 4, wq = pw % 4;
        const int j = lane % LP, q = lane / LP;
        const int nl = wq * NPW + q;                       // node within this CTA's share of the tile
        const int ch0 = j, ch1 = j + LP;                   // this lane's two 4-label chunks
        float cs[8];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            cs[u] = csum[4 * ch0 + u];
            cs[4 + u] = csum[4 * ch1 + u];
        }
        const unsigned stage_u = smem_u32(sB) + grp * S::STAGE_BYTES;
        float *iv = inv + grp * TC_N;
        const unsigned iv_remote = CG == 2 ? mapa(smem_u32(iv), rank ^ 1u) : 0u;
        long long i = grp;
        for (long long tile = cluster + grp * nclusters; tile < tiles;
             tile += TC_STAGES * nclusters, i += TC_STAGES) {
            const long long p0 = tile * TC_NODES;
            if (wq == 0 && lane < 5) {
                // the group's next tile: into L2 while this one is formed
                const long long np0 = p0 + (long long)TC_STAGES * nclusters * TC_NODES;
                if (np0 < npix && !(lane < 4 && a.first)) {
                    const long long n = npix - np0 < TC_NODES ? npix - np0 : TC_NODES;
                    const float *src = lane == 4
                        ? a.values + ((long long)(a.lr_begin - 1) * a.W + np0) * a.Ms
                        : a.msgs_in + lane * a.slot_stride + ((long long)a.lr_begin * a.W + np0) * a.Ms;
                    l2_prefetch(src, (unsigned)(n * a.Ms * 4));
                }
            }
            long long p = p0 + (long long)rank * S::NCTA + nl;
            const bool valid = p < npix;
            if (!valid) p = npix - 1;
            const int lr = a.lr_begin + (int)(p / a.W);
            const int c = (int)(p % a.W);
            const long long r = (long long)a.r0 + lr - 1;
            const long long node_l = (long long)lr * a.W + c;
            float g[8], m[4][8];
            {
                const float *gp = a.values + ((long long)(lr - 1) * a.W + c) * a.Ms;
                const float4 g0 = ldg_stream(reinterpret_cast<const float4 *>(gp + 4 * ch0));
                const float4 g1 = ldg_stream(reinterpret_cast<const float4 *>(gp + 4 * ch1));
                g[0] = g0.x; g[1] = g0.y; g[2] = g0.z; g[3] = g0.w;
                g[4] = g1.x; g[5] = g1.y; g[6] = g1.z; g[7] = g1.w;
                if (!a.first) {
                    const float *mp = a.msgs_in + node_l * a.Ms;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float4 m0 = ldg_stream(reinterpret_cast<const float4 *>(mp + k * a.slot_stride + 4 * ch0));
                        const float4 m1 = ldg_stream(reinterpret_cast<const float4 *>(mp + k * a.slot_stride + 4 * ch1));
                        m[k][0] = m0.x; m[k][1] = m0.y; m[k][2] = m0.z; m[k][3] = m0.w;
                        m[k][4] = m1.x; m[k][5] = m1.y; m[k][6] = m1.z; m[k][7] = m1.w;
                    }
                } else {
                    // bp.py:587-601 without touching memory
                    const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float real = ghost[k] ? 1.0f : 1.0f / (float)a.M;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int xx = u < 4 ? 4 * ch0 + u : 4 * ch1 + (u - 4);
                            m[k][u] = xx < a.M ? real : 0.0f;
                        }
                    }
                }
            }
            // the stage is free once the epilogue of the tile that used it is done
            bar_wait<CG>(&freeb[grp], (unsigned)(((i / TC_STAGES) & 1) ^ 1));
            const bool has[4] = {c + 1 < a.W, c > 0, r + 1 < a.H, r > 0};
            // exclusion products in the reference order (unary, then slots 0..3
            // ascending, skipping the excluded one; prefixes shared)
            float h[4][8], ab[8];
            vmul(h[3], g, m[1]);
            vmul(h[3], h[3], m[2]);
            vmul(h[3], h[3], m[3]);       // excl 0 -> dir 3
            vmul(ab, g, m[0]);
            vmul(h[1], ab, m[2]);
            vmul(h[1], h[1], m[3]);       // excl 1 -> dir 1
            vmul(ab, ab, m[1]);
            vmul(h[0], ab, m[3]);         // excl 2 -> dir 0
            vmul(h[2], ab, m[2]);         // excl 3 -> dir 2
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                const int row = nl * 4 + d;                // column of this CTA's h tile
                float hi[8], lo[8], sd = 0.0f;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    hi[u] = tf32_rna(h[d][u]);
                    lo[u] = h[d][u] - hi[u];
                    sd = fmaf(cs[u], h[d][u], sd);
                }
                const unsigned o0 = stage_u + sw128_chunk(row, ch0, S::B_ATOM);
                const unsigned o1 = stage_u + sw128_chunk(row, ch1, S::B_ATOM);
                sts128(o0, hi[0], hi[1], hi[2], hi[3]);
                sts128(o1, hi[4], hi[5], hi[6], hi[7]);
                sts128(o0 + S::B_PLANE, lo[0], lo[1], lo[2], lo[3]);
                sts128(o1 + S::B_PLANE, lo[4], lo[5], lo[6], lo[7]);
                sd = lanes_sum<LP>(sd);
                if (j == 0) {
                    const float rs = __frcp_rn(sd);
                    const int col = ((int)rank * S::NCTA + nl) * 4 + d;
                    iv[col] = rs;
                    if (CG == 2)
                        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(iv_remote + 4 * col), "f"(rs) : "memory");
                    const bool ok = (sd > 0.0f) && !isinf(sd);
                    if (!ok && valid && has[d])
                        report_failure(a.err, a.iteration, directed_edge_id(a.H, a.W, r, c, d));
                }
            }
            asm volatile("fence.proxy.async;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                bar_arrive<CG>(&full[grp], 0u);
                bar_arrive<CG>(&invf[grp], rank);
                if (CG == 2) bar_arrive<CG>(&invf[grp], rank ^ 1u);
            }
        }
    }

    // ---- teardown
    tc_fence_before();
    __syncthreads();
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (warp == TC_EPI_WARPS) {
        if (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(S::TCOLS) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(S::TCOLS) : "memory");
    }
}

template <int MS>
cudaError_t launch_dense_tc_ms(const DenseArgs &a, cudaStream_t s) {
    using S = TcShape<MS>;
    static int clusters_max = 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S::CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(TC_THREADS);
    cfg.dynamicSmemBytes = S::SMEM;
    cfg.stream = s;
    if (!clusters_max) {
        cudaError_t e = cudaFuncSetAttribute(dense_tc_kernel<MS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)S::SMEM);
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        clusters_max = sms / S::CG;
        if (S::CG > 1) {
            cfg.gridDim = dim3(sms);
            int n = 0;
            e = cudaOccupancyMaxActiveClusters(&n, dense_tc_kernel<MS>, &cfg);
            if (e != cudaSuccess) return e;
            if (n < 1) return cudaErrorLaunchOutOfResources;
            if (n < clusters_max) clusters_max = n;
        }
    }
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    long long clusters = (npix + TC_NODES - 1) / TC_NODES;
    if (clusters <= 0) return cudaSuccess;
    if (clusters > clusters_max) clusters = clusters_max;
    if (launch_block_cap() > 0 && clusters > launch_block_cap()) clusters = launch_block_cap();
    cfg.gridDim = dim3((unsigned)(clusters * S::CG));
    return cudaLaunchKernelEx(&cfg, dense_tc_kernel<MS>, a);
}

}  // namespace tc

bool dense_tc_supported(int Ms) { return Ms == 128 || Ms == 256; }

cudaError_t launch_dense_tc(const DenseArgs &a, cudaStream_t s) {
    switch (a.Ms) {
    case 128: return tc::launch_dense_tc_ms<128>(a, s);
    case 256: return tc::launch_dense_tc_ms<256>(a, s);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace sbp
