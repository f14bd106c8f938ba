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
// 2^-22 relative).  Variant C16 (SBP_DENSE_TC=2, opt-in) runs the two
// correction products in bf16 (kind::f16, K = 16 per MMA instead of 8) into
// the same accumulator: 64 instead of 96 MMAs per Ms = 256 tile, 2.47 vs
// 2.63 ms per C5 iteration, but 5.7e-6 instead of 3.2e-6 from the f64 oracle --
// too close to the 1e-5 bar to be the default.  Symmetric tables only (one resident copy serves both
// orientations), Ms = 128 (one CTA) or Ms = 256 (a CTA pair, cta_group::2,
// each CTA owning 128 of the 256 output labels).
//
// Tile shape.  On B200 one tcgen05.mma kind::tf32 (K = 8) takes >= 67 cycles
// whatever N <= 128 is (tools/tc_probe.cu mode 9, profiles/r02_tcgen05_mma_rate.txt:
// N = 32, 64, 128: 67 cycles; N = 256: 128), so the MMA N must be large: a
// tile is 24 nodes = 96 (node, direction) columns, the largest N whose
// operands fit beside the table.
//
// Per CTA:
//   tensor memory  columns [0, 96) and [128, 224): two accumulator stages
//                  [128 labels x 96 columns] fp32;
//                  Ms = 128: [256, 384) f_hi and [384, 512) f_lo rows of the table
//                  (both A operands from tensor memory, no shared-memory A reads);
//                  Ms = 256: [256, 512) f_lo, f_hi in shared memory
//   shared memory  Ms = 256: f_hi rows of this CTA [128 x 256] tf32, K-major,
//                  128-byte swizzle (128 KB);
//                  a ring of 48 KB slots, each one K-half (Ms/2 labels) of this
//                  CTA's columns of a tile, hi and lo planes, K-major swizzled
//                  (Ms = 128: 4 slots, Ms = 256: 2 slots)
// Warp roles (20 warps, one CTA per SM, persistent over tiles):
//   warps 0-3    epilogue: tcgen05.ld the accumulator (thread = output label),
//                scale by the column's 1/s, store into the neighbour's slot
//                (a warp stores 128 contiguous bytes per column)
//   warp 4       allocates tensor memory; one thread of the leader CTA issues
//                the tcgen05.mma of each K-half (3 products x Ms/16) and commits
//                to the slot's `empty` mbarrier (and the accumulator's `accf`)
//   warps 5-19   producers (5-18 in a CTA pair): read the unary and the four
//                incoming messages of their node(s) once, form the four
//                exclusion products in the reference order, split hi / lo
//                straight into the swizzled operand rows of the two K-half
//                slots, and compute the normaliser s = sum_{x_j} colsum_f(x_j)
//                h(x_j) (equal to the sum of the outputs up to rounding; the
//                reference divides by that sum).  Work items (tile, node slot)
//                are claimed from a shared-memory counter, so the twelve warps
//                run out of step and hide each other's load latency.
//   warp 19     (CTA pairs) relay: forwards the peer CTA's `full` arrivals to the
//                leader and copies this CTA's 1/s values to the other CTA, one
//                cluster-scope release fence per event instead of one per
//                producer warp and K-half
// mbarriers: full[slot] (producers -> MMA), empty[slot] (MMA commit -> producers),
// accf[stage] (MMA commit -> epilogue), accfree[stage] (epilogue -> MMA),
// linv[tile % 4] (producers -> epilogue / relay: the CTA's 1/s values),
// invf[tile % 4] (relay -> the other CTA's epilogue).
#include "aux_kernels.cuh"
#include "band_kernel.cuh"   // vmul, lanes_sum, smem_u32, mbar_init

namespace sbp {
namespace tc {

#ifdef SBP_TC_TRACE
// Debug build: cluster 0 records clock64 at the pipeline events of its first
// TRACE_TILES tiles (tools/tc_trace.py prints the timeline).
constexpr int TRACE_TILES = 48, TRACE_EVENTS = 16;
__device__ long long g_tc_trace[TRACE_TILES * TRACE_EVENTS];
#define TC_TRACE(tile_i, ev)                                                                    \
    do {                                                                                        \
        if (cluster == 0 && rank == 0 && lane == 0 && (tile_i) < TRACE_TILES)                   \
            g_tc_trace[(tile_i) * TRACE_EVENTS + (ev)] = clock64();                             \
    } while (0)
#else
#define TC_TRACE(tile_i, ev) do { } while (0)
#endif

constexpr int TC_NODES = 24;                // nodes per tile
constexpr int TC_N = 4 * TC_NODES;          // MMA N = 96: (node, direction) columns per tile
constexpr int TC_EPI_WARPS = 4;
constexpr int TC_ITEMS = 12;                // producer work items per tile and CTA
#ifndef SBP_TC_PROD_WARPS
#define SBP_TC_PROD_WARPS 15                // 20 warps: the register cap (96) is that of 17
#endif
constexpr int TC_PROD_WARPS = SBP_TC_PROD_WARPS;
constexpr int TC_WARPS = TC_EPI_WARPS + 1 + TC_PROD_WARPS;
constexpr int TC_THREADS = 32 * TC_WARPS;
constexpr int TC_ACC = 2;                   // accumulator stages, 128 tensor-memory columns apart
constexpr int TC_ACOL = 256;                // first tensor-memory column of the table operand(s)
constexpr int TC_TCOLS = 512;
constexpr int TC_INV = 4;                   // ring of per-tile 1/s vectors

template <int MS, bool C16 = false>
struct TcShape {
    static constexpr int CG = MS / 128;               // CTAs per MMA (cta_group)
    static constexpr int NB = TC_N / CG;              // tile columns (B rows) held by one CTA
    static constexpr int NCTA = TC_NODES / CG;        // nodes of a tile formed by one CTA
    static constexpr int LP = MS / 8;                 // lanes per node (8 labels each)
    static constexpr int NPW = 32 / LP;               // nodes per producer warp
    static constexpr int KH = MS / 2;                 // labels per K-half
    static constexpr int KSTEPS = KH / 8;             // tf32 MMAs (K = 8) per K-half: f_hi h_hi
    static constexpr int KSTEPS16 = KH / 16;          // bf16 MMAs (K = 16) per K-half and correction
    static constexpr int B_ATOM = NB * 128;           // bytes: NB rows x 32 tf32
    static constexpr int B_PLANE = (KH / 32) * B_ATOM;     // a tf32 plane (32 per 128-byte row): h_hi, h_lo
    static constexpr int B_PLANE16 = (KH / 64) * B_ATOM;   // C16: bf16 planes (64 per row): bf16(h), bf16(h_lo)
    static constexpr int SLOT_BYTES = 2 * B_PLANE;         // 48 KB either way (2 B_PLANE16 = B_PLANE)
    static constexpr int NSLOT = MS == 128 ? 4 : 2;
    static constexpr bool A_HI_SMEM = MS == 256;      // f_hi in shared memory (no room in tensor memory)
    static constexpr int A_ATOM = 128 * 128;          // bytes: 128 rows x 32 tf32
    static constexpr int A_BYTES = A_HI_SMEM ? (MS / 32) * A_ATOM : 0;
    // tensor-memory columns of the table operands: f_hi as tf32 (Ms = 128 only,
    // one column per k), then f_lo as tf32 -- or, C16, bf16(f_lo) and bf16(f),
    // two k per column
    static constexpr int ACOL_HI = TC_ACOL;
    static constexpr int ACOL_LO = MS == 128 ? TC_ACOL + 128 : TC_ACOL;
    static constexpr int ACOL_LO16 = ACOL_LO;
    static constexpr int ACOL_HI16 = ACOL_LO16 + MS / 2;
    static_assert(ACOL_LO + MS <= TC_TCOLS, "tensor-memory budget");
    static constexpr int RELAY = CG == 2 ? 1 : 0;     // pairs: the last warp relays, 14 produce
    static constexpr int THREADS = TC_THREADS;        // 640: more threads would cap registers at 80
    static constexpr int AUX_BYTES = 3072;            // colsum, 1/s ring, mbarriers, tmem address
    static constexpr size_t SMEM = (size_t)A_BYTES + NSLOT * SLOT_BYTES + AUX_BYTES;
    static_assert(MS == 128 || MS == 256, "tensor-core dense kernel: Ms = 128 or 256");
    static_assert(NPW * TC_ITEMS == NCTA, "an item is one producer-warp pass: NPW nodes");
    static_assert(SLOT_BYTES == 49152 && SMEM <= 232448, "shared-memory budget");
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

__device__ __forceinline__ void bar_arrive_relaxed(unsigned long long *bar, unsigned rank) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa(smem_u32(bar), rank)) : "memory");
}

// Wait on an mbarrier phase.  try_wait suspends the thread in hardware for up
// to the time hint, so waiting warps take no issue slots from working ones
// (a polling loop did: 40 % of the executed instructions were polls).  Bounded:
// a protocol error traps instead of hanging the device.
template <int CG, int SLEEP>
__device__ __forceinline__ void bar_wait(unsigned long long *bar, unsigned parity) {
    unsigned done = 0;
    for (unsigned spin = 0; !done; ++spin) {
        if (CG == 1)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n"
                         " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity), "r"(20000u) : "memory");
        else
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n"
                         " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity), "r"(20000u) : "memory");
        if (spin > (1u << 24)) __trap();
    }
}

__device__ __forceinline__ bool elect_one() {
    unsigned pred;
    asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void st_global_if(float *p, float v, bool pred) {
    asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f32 [%0], %1;\n}" ::"l"(p), "f"(v),
                 "r"((int)pred) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Round to tf32 (10 explicit mantissa bits), nearest with ties away from zero,
// on the bit pattern: add half a tf32 ulp and clear the 13 low bits.  Finite
// non-negative inputs (tables and products of probabilities); cvt.rna.tf32.f32
// compiles to a five-instruction sequence on sm_100a.
__device__ __forceinline__ float tf32_rna(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
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

// kind::f16 with bf16 operands (A: two k per tensor-memory column), same fp32 accumulator
template <int CG>
__device__ __forceinline__ void mma_ts16(unsigned d, unsigned a_tmem, unsigned long long b, unsigned idesc,
                                         unsigned acc) {
    if (CG == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem),
                     "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem),
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

// two floats -> one 32-bit word of bf16 (a in the low half: the lower k / label)
__device__ __forceinline__ float pack_bf16(float a, float b) {
    unsigned r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
    return __uint_as_float(r);
}

__device__ __forceinline__ void sts64(unsigned saddr, float a, float b) {
    asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(saddr), "f"(a), "f"(b) : "memory");
}

// (o0, o1) += (a0 * b0, a1 * b1)
__device__ __forceinline__ void fma2v(float &o0, float &o1, float a0, float a1, float b0, float b1) {
    unsigned long long r = f2_pack(o0, o1);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(f2_pack(a0, a1)), "l"(f2_pack(b0, b1)));
    f2_unpack(r, o0, o1);
}

__device__ __forceinline__ void sts128(unsigned saddr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// ---- the kernel --------------------------------------------------------------

template <int MS, bool C16>
__global__ void __launch_bounds__(TcShape<MS, C16>::THREADS, 1)
dense_tc_kernel(const __grid_constant__ DenseArgs a) {
    using S = TcShape<MS, C16>;
    constexpr int CG = S::CG;
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    unsigned char *sA = tc_smem;                       // Ms = 256: f_hi
    unsigned char *sB = tc_smem + S::A_BYTES;          // slot ring
    float *csum = reinterpret_cast<float *>(sB + S::NSLOT * S::SLOT_BYTES);   // [MS]
    float *inv = csum + MS;                                                   // [TC_INV][TC_N]
    unsigned long long *bars = reinterpret_cast<unsigned long long *>(inv + TC_INV * TC_N);
    // `empty` has two generations per slot: a parity wait cannot tell phase k
    // from phase k + 2, and a producer that claimed an item early can be two
    // uses of a slot ahead of the MMA (it overwrote live operand rows once);
    // with use u on barrier [slot + NSLOT (u % 2)] the alias is four uses away,
    // further than the item counter lets any warp run ahead.
    unsigned long long *full = bars, *empty = bars + 4, *accf = bars + 12, *accfree = bars + 14,
                       *invf = bars + 16, *linv = bars + 20;
    unsigned *tmem_slot = reinterpret_cast<unsigned *>(bars + 24);
    unsigned *item_ctr = tmem_slot + 1;                // producers' work-item counter

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned rank = CG == 2 ? cluster_rank() : 0u;
    const long long cluster = blockIdx.x / CG, nclusters = gridDim.x / CG;
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long tiles = (npix + TC_NODES - 1) / TC_NODES;
    const float *tab = a.t[0];

    // ---- one-time setup: table operands, column sums, barriers, tensor memory
    if (S::A_HI_SMEM) {
        for (int i = tid; i < 128 * (MS / 4); i += S::THREADS) {
            const int row = i / (MS / 4), ch = i % (MS / 4);
            const float4 v = *reinterpret_cast<const float4 *>(tab + (size_t)(128 * rank + row) * MS + 4 * ch);
            sts128(smem_u32(sA) + sw128_chunk(row, ch, S::A_ATOM), tf32_rna(v.x), tf32_rna(v.y),
                   tf32_rna(v.z), tf32_rna(v.w));
        }
    }
    {
        // column sums of the whole table, fixed order: SL row slices, then the slices
        constexpr int SL = 2;
        float *part = reinterpret_cast<float *>(sB);   // [SL][MS] scratch in slot 0
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
        for (int s = 0; s < S::NSLOT; ++s) {
            // the leader's `full` counts its own producers' items and, in a
            // pair, one forwarded arrival from the peer's relay warp
            mbar_init(&full[s], TC_ITEMS + (CG == 2 && rank == 0 ? 1 : 0));
            mbar_init(&empty[s], 1);
            mbar_init(&empty[s + S::NSLOT], 1);
        }
        for (int s = 0; s < TC_ACC; ++s) {
            mbar_init(&accf[s], 1);
            mbar_init(&accfree[s], TC_EPI_WARPS * CG);
        }
        for (int s = 0; s < TC_INV; ++s) {
            mbar_init(&linv[s], TC_ITEMS);   // this CTA's producers: their 1/s values are written
            mbar_init(&invf[s], 1);          // pair: the peer's relay has copied its half over
        }
        *item_ctr = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == TC_EPI_WARPS) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)), "n"(TC_TCOLS) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)), "n"(TC_TCOLS) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tmem = *tmem_slot;
    if (warp < TC_EPI_WARPS) {
        // table rows of this CTA -> tensor memory: lane = label row, column = k
        const float *row = tab + (size_t)(128 * rank + 32 * warp + lane) * MS;
        const unsigned lane_base = tmem + ((unsigned)(32 * warp) << 16);
        if constexpr (C16) {
            for (int k0 = 0; k0 < MS; k0 += 64) {
                float lo16[32], hi16[32];   // packed bf16 pairs: columns (k0 / 2) .. + 31
    #pragma unroll
                for (int half = 0; half < 2; ++half) {
                    float hi[32];
    #pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const float2 t = *reinterpret_cast<const float2 *>(row + k0 + 32 * half + i);
                        hi[i] = tf32_rna(t.x);
                        hi[i + 1] = tf32_rna(t.y);
                        lo16[16 * half + i / 2] = pack_bf16(t.x - hi[i], t.y - hi[i + 1]);
                        hi16[16 * half + i / 2] = pack_bf16(t.x, t.y);
                    }
                    if (!S::A_HI_SMEM) tmem_st32(lane_base + S::ACOL_HI + k0 + 32 * half, hi);
                }
                tmem_st32(lane_base + S::ACOL_LO16 + k0 / 2, lo16);
                tmem_st32(lane_base + S::ACOL_HI16 + k0 / 2, hi16);
            }
        } else {
            for (int k0 = 0; k0 < MS; k0 += 32) {
                float hi[32], lo[32];
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    const float4 t = *reinterpret_cast<const float4 *>(row + k0 + i);
                    hi[i] = tf32_rna(t.x); hi[i + 1] = tf32_rna(t.y);
                    hi[i + 2] = tf32_rna(t.z); hi[i + 3] = tf32_rna(t.w);
                    lo[i] = t.x - hi[i]; lo[i + 1] = t.y - hi[i + 1];
                    lo[i + 2] = t.z - hi[i + 2]; lo[i + 3] = t.w - hi[i + 3];
                }
                if (!S::A_HI_SMEM) tmem_st32(lane_base + S::ACOL_HI + k0, hi);
                tmem_st32(lane_base + S::ACOL_LO + k0, lo);
            }
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
        // Thread = output label x; column n = (node, direction).  The four
        // destinations of a node are fixed offsets from the node's own slot-0
        // address, and consecutive nodes of a tile are consecutive in memory.
        const int x = 128 * (int)rank + 32 * warp + lane;
        const long long W = a.W;
        float *const d0 = a.msgs_out + x + dir_wslot(0) * a.slot_stride + a.Ms;       // right neighbour
        float *const d1 = a.msgs_out + x + dir_wslot(1) * a.slot_stride - a.Ms;       // left
        float *const d2 = a.msgs_out + x + dir_wslot(2) * a.slot_stride + W * a.Ms;   // below
        float *const d3 = a.msgs_out + x + dir_wslot(3) * a.slot_stride - W * a.Ms;   // above
        long long i = 0;
        for (long long tile = cluster; tile < tiles; tile += nclusters, ++i) {
            const int acc = (int)(i % TC_ACC), ir = (int)(i % TC_INV);
            bar_wait<1, 0>(&linv[ir], (unsigned)((i / TC_INV) & 1));
            if (CG == 2) bar_wait<CG, 0>(&invf[ir], (unsigned)((i / TC_INV) & 1));
            bar_wait<CG, 0>(&accf[acc], (unsigned)((i / TC_ACC) & 1));
            tc_fence_after();
            if (warp == 0) TC_TRACE(i, 0);
            const float4 *iv4 = reinterpret_cast<const float4 *>(inv + ir * TC_N);
            const long long p0 = tile * TC_NODES;
            const unsigned lq = (unsigned)p0 / (unsigned)a.W;
            int lr = a.lr_begin + (int)lq;
            int c = (int)((unsigned)p0 - lq * (unsigned)a.W);
            long long off = ((long long)lr * W + c) * a.Ms;   // node's element offset in a slot plane
            long long left = npix - p0;                        // nodes of the strip from p0 on
#pragma unroll 1
            for (int cc = 0; cc < TC_N / 32; ++cc) {
                float v[32];
                float4 s4[8];
#pragma unroll
                for (int n = 0; n < 8; ++n) s4[n] = iv4[8 * cc + n];   // the 1/s of 8 nodes (broadcast reads)
                tmem_ld32(tmem + ((unsigned)(32 * warp) << 16) + 128 * acc + 32 * cc, v);
#pragma unroll
                for (int n = 0; n < 8; ++n) {
                    const bool in = left > 0;
                    const long long r = (long long)a.r0 + lr - 1;
                    st_global_if(d0 + off, v[4 * n + 0] * s4[n].x, in && c + 1 < a.W);
                    st_global_if(d1 + off, v[4 * n + 1] * s4[n].y, in && c > 0);
                    st_global_if(d2 + off, v[4 * n + 2] * s4[n].z, in && r + 1 < a.H);
                    st_global_if(d3 + off, v[4 * n + 3] * s4[n].w, in && r > 0);
                    off += a.Ms;
                    --left;
                    if (++c == a.W) { c = 0; ++lr; }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {                                    // the leader's MMA thread waits on it
                if (rank == 0) bar_arrive<1>(&accfree[acc], 0u);
                else bar_arrive<CG>(&accfree[acc], 0u);
            }
            if (warp == 0) TC_TRACE(i, 1);
        }
    } else if (warp == TC_EPI_WARPS) {
        // ================= MMA issuer (leader CTA) =================
        // The whole warp runs this code with warp-uniform values (descriptors
        // stay in the uniform datapath); one elected lane issues.
        if (rank == 0) {
            const unsigned mn = ((unsigned)(TC_N >> 3) << 17) | ((unsigned)((128 * CG) >> 4) << 24);
            const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | mn;     // tf32 x tf32 -> f32
            const unsigned idesc16 = (1u << 4) | (1u << 7) | (1u << 10) | mn;   // bf16 x bf16 -> f32
            const unsigned long long a_desc0 = sw128_desc(smem_u32(sA));
            const unsigned sB_u = smem_u32(sB);
            long long i = 0;
            for (long long tile = cluster; tile < tiles; tile += nclusters, ++i) {
                const int acc = (int)(i % TC_ACC);
                bar_wait<CG, 0>(&accfree[acc], (unsigned)(((i / TC_ACC) & 1) ^ 1));
                TC_TRACE(i, 2);
                const unsigned d = tmem + 128 * acc;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const long long q = 2 * i + hh;
                    const int slot = (int)(q % S::NSLOT);
                    bar_wait<CG, 0>(&full[slot], (unsigned)((q / S::NSLOT) & 1));
                    tc_fence_after();
                    TC_TRACE(i, 3 + 2 * hh);
                    const unsigned long long bhi = sw128_desc(sB_u + slot * S::SLOT_BYTES);
                    const unsigned long long blo = bhi + (S::B_PLANE >> 4);      // h_lo (tf32), or, C16:
                    const unsigned long long bhi16 = blo;                          // bf16(h), then bf16(h_lo)
                    const unsigned long long blo16 = bhi16 + (S::B_PLANE16 >> 4);
                    if (elect_one()) {
                        // corrections first (small terms), then f_hi h_hi, all into one fp32
                        // accumulator; descriptor offsets are compile-time constants (>> 4:
                        // 16-byte units)
                        if constexpr (C16) {
#pragma unroll
                            for (int k = 0; k < S::KSTEPS16; ++k) {         // bf16(f_lo) bf16(h)
                                const int kk = hh * S::KSTEPS16 + k;
                                mma_ts16<CG>(d, tmem + S::ACOL_LO16 + 8 * kk,
                                             bhi16 + (((k >> 2) * S::B_ATOM + (k & 3) * 32) >> 4), idesc16,
                                             (hh | k) > 0);
                            }
#pragma unroll
                            for (int k = 0; k < S::KSTEPS16; ++k) {         // bf16(f) bf16(h_lo)
                                const int kk = hh * S::KSTEPS16 + k;
                                mma_ts16<CG>(d, tmem + S::ACOL_HI16 + 8 * kk,
                                             blo16 + (((k >> 2) * S::B_ATOM + (k & 3) * 32) >> 4), idesc16, 1u);
                            }
                        } else {
#pragma unroll
                            for (int k = 0; k < S::KSTEPS; ++k) {           // f_hi h_lo
                                const int kk = hh * S::KSTEPS + k;
                                const unsigned long long bd = blo + (((k >> 2) * S::B_ATOM + (k & 3) * 32) >> 4);
                                if (S::A_HI_SMEM)
                                    mma_ss<CG>(d, a_desc0 + (((kk >> 2) * S::A_ATOM + (kk & 3) * 32) >> 4), bd,
                                               idesc, (hh | k) > 0);
                                else
                                    mma_ts<CG>(d, tmem + S::ACOL_HI + 8 * kk, bd, idesc, (hh | k) > 0);
                            }
#pragma unroll
                            for (int k = 0; k < S::KSTEPS; ++k) {           // f_lo h_hi
                                const int kk = hh * S::KSTEPS + k;
                                mma_ts<CG>(d, tmem + S::ACOL_LO + 8 * kk,
                                           bhi + (((k >> 2) * S::B_ATOM + (k & 3) * 32) >> 4), idesc, 1u);
                            }
                        }
#pragma unroll
                        for (int k = 0; k < S::KSTEPS; ++k) {               // f_hi h_hi
                            const int kk = hh * S::KSTEPS + k;
                            const unsigned long long bd = bhi + (((k >> 2) * S::B_ATOM + (k & 3) * 32) >> 4);
                            if (S::A_HI_SMEM)
                                mma_ss<CG>(d, a_desc0 + (((kk >> 2) * S::A_ATOM + (kk & 3) * 32) >> 4), bd, idesc, 1u);
                            else
                                mma_ts<CG>(d, tmem + S::ACOL_HI + 8 * kk, bd, idesc, 1u);
                        }
                        // the slot is free once these complete: use u of the slot, generation u % 2
                        mma_commit<CG>(&empty[slot + S::NSLOT * (int)((q / S::NSLOT) & 1)]);
                        if (hh == 1) mma_commit<CG>(&accf[acc]);
                    }
                    __syncwarp();
                    TC_TRACE(i, 4 + 2 * hh);
                }
            }
        }
    } else if (S::RELAY && warp == TC_WARPS - 1) {
        // ================= relay (CTA pairs) =================
        // Forwards this CTA's producer progress to the peer with ONE
        // cluster-scope release per event: the peer CTA's `full` arrivals to
        // the leader's barrier, and this CTA's half of the 1/s vector to the
        // other CTA's epilogue.
        long long i = 0;
        for (long long tile = cluster; tile < tiles; tile += nclusters, ++i) {
            const int ir = (int)(i % TC_INV);
            if (rank == 1) {
                const long long q0 = 2 * i;
                const int s0 = (int)(q0 % S::NSLOT);
                bar_wait<1, 0>(&full[s0], (unsigned)((q0 / S::NSLOT) & 1));
                if (lane == 0) {
                    asm volatile("fence.acq_rel.cluster;" ::: "memory");
                    bar_arrive_relaxed(&full[s0], 0u);
                }
                const long long q1 = q0 + 1;
                const int s1 = (int)(q1 % S::NSLOT);
                bar_wait<1, 0>(&full[s1], (unsigned)((q1 / S::NSLOT) & 1));
            }
            bar_wait<1, 0>(&linv[ir], (unsigned)((i / TC_INV) & 1));
            float *mine = inv + ir * TC_N + (int)rank * S::NB;
            for (int c = lane; c < S::NB; c += 32)
                asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(mapa(smem_u32(mine + c), rank ^ 1u)),
                             "f"(mine[c]) : "memory");
            __syncwarp();
            if (lane == 0) {
                asm volatile("fence.acq_rel.cluster;" ::: "memory");
                if (rank == 1) bar_arrive_relaxed(&full[(int)((2 * i + 1) % S::NSLOT)], 0u);
                bar_arrive_relaxed(&invf[ir], rank ^ 1u);
            }
            __syncwarp();
        }
    } else {
        // ================= producers =================
        constexpr int LP = S::LP, NPW = S::NPW;
        // Work items are claimed from a per-CTA counter: item = (tile sequence
        // number i, node slot pw of the tile).  Identical warps run at different
        // speeds (they share schedulers with the MMA and epilogue warps), and a
        // static warp -> node map made every tile wait for the slowest one.
        const int j = lane % LP, q = lane / LP;
        const unsigned sB_u = smem_u32(sB);
        float g[8], m[4][8];
        long long p, node_l, r;
        int c, nl;
        bool valid;
        auto claim = [&]() -> unsigned {
            unsigned it = 0;
            if (lane == 0) it = atomicAdd(item_ctr, 1u);
            return __shfl_sync(SBP_FULL_MASK, it, 0);
        };
        auto locate = [&](long long tile, int pw) {
            nl = pw * NPW + q;                             // node within this CTA's share of the tile
            p = tile * TC_NODES + (long long)rank * S::NCTA + nl;
            valid = p < npix;
            if (!valid) p = npix - 1;
            const unsigned lq = (unsigned)p / (unsigned)a.W;      // strips hold < 2^31 nodes (launcher)
            const int lr = a.lr_begin + (int)lq;
            c = (int)((unsigned)p - lq * (unsigned)a.W);
            r = (long long)a.r0 + lr - 1;
            node_l = (long long)lr * a.W + c;
        };
        auto load = [&]() {
            const float *gp = a.values + (node_l - a.W) * a.Ms;   // values row lr - 1
            const float4 g0 = ldg_stream(reinterpret_cast<const float4 *>(gp + 4 * j));
            const float4 g1 = ldg_stream(reinterpret_cast<const float4 *>(gp + S::KH + 4 * j));
            g[0] = g0.x; g[1] = g0.y; g[2] = g0.z; g[3] = g0.w;
            g[4] = g1.x; g[5] = g1.y; g[6] = g1.z; g[7] = g1.w;
            if (!a.first) {
                const float *mp = a.msgs_in + node_l * a.Ms;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float4 m0 = ldg_stream(reinterpret_cast<const float4 *>(mp + k * a.slot_stride + 4 * j));
                    const float4 m1 = ldg_stream(reinterpret_cast<const float4 *>(mp + k * a.slot_stride + S::KH + 4 * j));
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
                        const int xx = u < 4 ? 4 * j + u : S::KH + 4 * j + (u - 4);
                        m[k][u] = xx < a.M ? real : 0.0f;
                    }
                }
            }
        };
        // No loads stay in flight across the publishing fences / release
        // arrives (they would wait for them, and the compiler spilled the
        // in-flight registers): a warp exposes its own load latency, and the
        // twelve warps, out of step through the item counter, hide each other's.
        while (true) {
            const unsigned item = claim();
            const long long i = item / TC_ITEMS;
            const int pw = (int)(item % TC_ITEMS);
            const long long tile = cluster + i * nclusters;
            if (tile >= tiles) break;
            locate(tile, pw);
            load();
            if (pw == 0) TC_TRACE(i, 7);
            const int nl_cur = nl;
            // this lane's 16-byte chunk (4 tf32) and 8-byte half chunk (4 bf16) of its node's four rows
            unsigned row_off[4], row_off16[4];
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                row_off[d] = (unsigned)sw128_chunk(nl_cur * 4 + d, j, S::B_ATOM);
                row_off16[d] = (unsigned)sw128_chunk(nl_cur * 4 + d, j >> 1, S::B_ATOM) + (j & 1) * 8;
            }
            const long long r_cur = r;
            const int c_cur = c;
            const bool valid_cur = valid;
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
            if (pw == 0) TC_TRACE(i, 8);
            const long long i_cur = i;
            const int pw_cur = pw;
            float sd[4][2] = {{0.0f, 0.0f}, {0.0f, 0.0f}, {0.0f, 0.0f}, {0.0f, 0.0f}};
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const long long qq = 2 * i_cur + hh;
                const int slot = (int)(qq % S::NSLOT);
                const long long use = qq / S::NSLOT;           // this is the use-th fill of the slot
                if (use > 0)                                   // wait for the MMAs of fill use - 1
                    bar_wait<CG, 64>(&empty[slot + S::NSLOT * (int)((use - 1) & 1)],
                                     (unsigned)(((use - 1) >> 1) & 1));
                if (pw_cur == 0) TC_TRACE(i_cur, 9 + 2 * hh);
                const unsigned slot_u = sB_u + slot * S::SLOT_BYTES;
                const float4 cs4 = *reinterpret_cast<const float4 *>(csum + hh * S::KH + 4 * j);
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    const float *hv = &h[d][4 * hh];
                    float hi[4], lo[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) hi[u] = tf32_rna(hv[u]);
                    sub2(lo[0], lo[1], hv[0], hv[1], hi[0], hi[1]);
                    sub2(lo[2], lo[3], hv[2], hv[3], hi[2], hi[3]);
                    // normaliser partial sums (two lanes of a packed accumulator per direction)
                    fma2v(sd[d][0], sd[d][1], cs4.x, cs4.y, hv[0], hv[1]);
                    fma2v(sd[d][0], sd[d][1], cs4.z, cs4.w, hv[2], hv[3]);
                    sts128(slot_u + row_off[d], hi[0], hi[1], hi[2], hi[3]);
                    if constexpr (C16) {
                        const unsigned o16 = slot_u + S::B_PLANE + row_off16[d];
                        sts64(o16, pack_bf16(hv[0], hv[1]), pack_bf16(hv[2], hv[3]));
                        sts64(o16 + S::B_PLANE16, pack_bf16(lo[0], lo[1]), pack_bf16(lo[2], lo[3]));
                    } else {
                        sts128(slot_u + S::B_PLANE + row_off[d], lo[0], lo[1], lo[2], lo[3]);
                    }
                }
                if (hh == 1) {
                    // 1/s of the node's four messages, before the slot is published
                    const int ir = (int)(i_cur % TC_INV);
                    float *iv = inv + ir * TC_N;
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        const float s = lanes_sum<LP>(sd[d][0] + sd[d][1]);
                        if (j == 0) {
                            const float rs = __frcp_rn(s);
                            const int col = ((int)rank * S::NCTA + nl_cur) * 4 + d;
                            iv[col] = rs;               // a pair's relay warp copies it to the peer
                            const bool ok = (s > 0.0f) && !isinf(s);
                            if (!ok && valid_cur && has[d])
                                report_failure(a.err, a.iteration, directed_edge_id(a.H, a.W, r_cur, c_cur, d));
                        }
                    }
                }
                // this thread's operand rows (generic proxy, own shared memory) -> tensor-core reads
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    // CTA-scope releases only: in a pair the relay warp forwards
                    // (a cluster-scope fence here cost ~1500 cycles per half and warp)
                    bar_arrive<1>(&full[slot], 0u);
                    if (hh == 1) bar_arrive<1>(&linv[(int)(i_cur % TC_INV)], 0u);
                }
                if (pw_cur == 0) TC_TRACE(i_cur, 10 + 2 * hh);
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
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TCOLS) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TCOLS) : "memory");
    }
}

template <int MS, bool C16>
cudaError_t launch_dense_tc_ms(const DenseArgs &a, cudaStream_t s) {
    using S = TcShape<MS, C16>;
    static int clusters_max = 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S::CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(S::THREADS);
    cfg.dynamicSmemBytes = S::SMEM;
    cfg.stream = s;
    if (!clusters_max) {
        cudaError_t e = cudaFuncSetAttribute(dense_tc_kernel<MS, C16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)S::SMEM);
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        clusters_max = sms / S::CG;
        if (S::CG > 1) {
            cfg.gridDim = dim3(sms);
            int n = 0;
            e = cudaOccupancyMaxActiveClusters(&n, dense_tc_kernel<MS, C16>, &cfg);
            if (e != cudaSuccess) return e;
            if (n < 1) return cudaErrorLaunchOutOfResources;
            if (n < clusters_max) clusters_max = n;
        }
    }
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    if (npix >= (1ll << 31)) return cudaErrorNotSupported;   // 32-bit node coordinates in the kernel
    long long clusters = (npix + TC_NODES - 1) / TC_NODES;
    if (clusters <= 0) return cudaSuccess;
    if (clusters > clusters_max) clusters = clusters_max;
    if (launch_block_cap() > 0 && clusters > launch_block_cap()) clusters = launch_block_cap();
    cfg.gridDim = dim3((unsigned)(clusters * S::CG));
    return cudaLaunchKernelEx(&cfg, dense_tc_kernel<MS, C16>, a);
}

}  // namespace tc

bool dense_tc_supported(int Ms) { return Ms == 128 || Ms == 256; }

#ifdef SBP_TC_TRACE
}  // namespace sbp
extern "C" __attribute__((visibility("default"))) int sbp_debug_tc_trace(long long *out, int n) {
    const int total = sbp::tc::TRACE_TILES * sbp::tc::TRACE_EVENTS;
    if (n > total) n = total;
    cudaDeviceSynchronize();
    return (int)cudaMemcpyFromSymbol(out, sbp::tc::g_tc_trace, sizeof(long long) * n);
}
namespace sbp {
#endif

cudaError_t launch_dense_tc(const DenseArgs &a, bool bf16_corrections, cudaStream_t s) {
    switch (a.Ms) {
    case 128: return bf16_corrections ? tc::launch_dense_tc_ms<128, true>(a, s) : tc::launch_dense_tc_ms<128, false>(a, s);
    case 256: return bf16_corrections ? tc::launch_dense_tc_ms<256, true>(a, s) : tc::launch_dense_tc_ms<256, false>(a, s);
    default: return cudaErrorNotSupported;
    }
}

}  // namespace sbp
