// tcgen05 probe: validates, on a B200, the operand layouts the tensor-core
// dense kernel (dense_tc_kernel.cu) relies on, before that kernel is trusted:
//   mode 0  cta_group::1, A and B from shared memory (K-major, 128-byte swizzle)
//   mode 1  cta_group::1, A from tensor memory (lane = row, column = k), B smem
//   mode 2  cta_group::2 (CTA pair, M = 256), A and B from shared memory
//   mode 3  cta_group::2, A from tensor memory
//   mode 4/5  kind::tf32 and kind::f16 (bf16, A packed two per tensor-memory column)
//           products accumulated into one accumulator, cta_group::1 / ::2
//   mode 9  MMA issue rate against N, SS / TS, cta_group
// D[M x N] = A[M x K] * B[N x K]^T in kind::tf32, compared on the host with an
// f64 product of the tf32-truncated inputs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tc_probe tools/tc_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ bool mbar_wait(unsigned long long *bar, unsigned parity) {
    unsigned done = 0;
    for (long long spin = 0; !done; ++spin) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (spin > (1ll << 24)) return false;
    }
    return true;
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm_100 version 1):
// rows of 128 bytes (32 tf32), 8-row groups 1024 bytes apart (SBO), the 16-byte
// chunk c of row r stored at chunk c ^ (r % 8).
__device__ __forceinline__ unsigned long long sw128_desc(unsigned saddr) {
    return (unsigned long long)((saddr & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ unsigned sw128_off(int row, int k, int atom_bytes) {
    const int ka = k >> 5, c = (k & 31) >> 2;
    return ka * atom_bytes + (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4) + (k & 3) * 4;
}

template <int CG>
__device__ __forceinline__ void mma_ss(unsigned d, unsigned long long a, unsigned long long b, unsigned idesc, unsigned acc) {
    if (CG == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
template <int CG>
__device__ __forceinline__ void mma_ts(unsigned d, unsigned a_tmem, unsigned long long b, unsigned idesc, unsigned acc) {
    if (CG == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__device__ __forceinline__ void tmem_ld32(unsigned taddr, float (&v)[32]) {
    unsigned r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st32(unsigned taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(taddr),
          "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
          "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
          "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
          "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])),
          "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
          "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
          "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])),
          "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
        : "memory");
}

constexpr int K = 128;       // 4 swizzle atoms, 16 MMAs of K = 8
constexpr int N = 32;
constexpr int TCOLS = 256;   // tensor-memory columns: [0, N) accumulator, [128, 128 + K) A operand

// CG = 1: one CTA, M = 128.  CG = 2: a CTA pair, M = 256 (128 rows per CTA), B split by N halves.
template <int CG, bool ATMEM>
__global__ void __launch_bounds__(128) probe(const float *A, const float *B, float *D, int *status) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    unsigned rank = 0;
    if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    constexpr int NB = N / CG;                 // B rows held by this CTA
    constexpr int A_ATOM = 128 * 128, B_ATOM = NB * 128;
    unsigned char *sA = smem, *sB = smem + (K / 32) * A_ATOM;
    const float *Ar = A + (size_t)rank * 128 * K;
    const float *Br = B + (size_t)rank * NB * K;
    if (!ATMEM)
        for (int i = tid; i < 128 * K; i += 128)
            *(float *)(sA + sw128_off(i / K, i % K, A_ATOM)) = Ar[i];
    for (int i = tid; i < NB * K; i += 128)
        *(float *)(sB + sw128_off(i / K, i % K, B_ATOM)) = Br[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)), "n"(TCOLS) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)), "n"(TCOLS) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base_s;
    if (ATMEM) {
        // row (32 warp + lane) of this CTA's A half -> lane, k -> column 128 + k
        for (int k0 = 0; k0 < K; k0 += 32) {
            float v[32];
            for (int i = 0; i < 32; ++i) v[i] = Ar[(size_t)(32 * warp + lane) * K + k0 + i];
            tmem_st32(tmem + ((unsigned)(32 * warp) << 16) + 128 + k0, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (tid == 0 && rank == 0) {
        const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(N >> 3) << 17) |
                               ((unsigned)((128 * CG) >> 4) << 24);
        for (int k = 0; k < K / 8; ++k) {
            const int ka = k >> 2, ks = k & 3;
            const unsigned long long bd = sw128_desc(smem_u32(sB) + ka * B_ATOM + ks * 32);
            if (ATMEM) {
                mma_ts<CG>(tmem, tmem + 128 + 8 * k, bd, idesc, k > 0);
            } else {
                const unsigned long long ad = sw128_desc(smem_u32(sA) + ka * A_ATOM + ks * 32);
                mma_ss<CG>(tmem, ad, bd, idesc, k > 0);
            }
        }
        if (CG == 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((unsigned short)3) : "memory");
    }
    const bool ok = mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (!ok) {
        if (tid == 0) status[rank] = 1;
    } else {
        float v[32];
        tmem_ld32(tmem + ((unsigned)(32 * warp) << 16), v);
        for (int j = 0; j < N; ++j) D[((size_t)rank * 128 + 32 * warp + lane) * N + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (warp == 0) {
        if (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TCOLS) : "memory");
    }
}

static float tf32_trunc(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    memcpy(&x, &u, 4);
    return x;
}

template <int CG, bool ATMEM>
static int run(const char *name) {
    const int M = 128 * CG;
    std::vector<float> A((size_t)M * K), B((size_t)N * K), D((size_t)M * N, -1.0f);
    srand(1234);
    for (auto &x : A) x = tf32_trunc((float)rand() / RAND_MAX + 0.01f);
    for (auto &x : B) x = tf32_trunc((float)rand() / RAND_MAX - 0.3f);
    float *dA, *dB, *dD;
    int *dS, hS[2] = {0, 0};
    CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
    CK(cudaMalloc(&dS, 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dD, D.data(), D.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dS, 0, 8));
    const size_t smem = (K / 32) * (128 * 128) + (K / 32) * (N / CG * 128);
    CK(cudaFuncSetAttribute(probe<CG, ATMEM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CG); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, probe<CG, ATMEM>, (const float *)dA, (const float *)dB, dD, dS));
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: kernel failed: %s\n", name, cudaGetErrorString(e)); return 2; }
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hS, dS, 8, cudaMemcpyDeviceToHost));
    double worst = 0.0; int bad = 0, fi = -1, fj = -1;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double ref = 0.0;
            for (int k = 0; k < K; ++k) ref += (double)A[(size_t)i * K + k] * (double)B[(size_t)j * K + k];
            const double err = fabs(ref - D[(size_t)i * N + j]) / (fabs(ref) + 1.0);
            if (err > worst) worst = err;
            if (err > 1e-4) { if (!bad) { fi = i; fj = j; } ++bad; }
        }
    printf("%s: timeout flags %d %d, worst rel err %.3e, bad %d of %d (first bad %d,%d: got %g)\n", name, hS[0], hS[1],
           worst, bad, M * N, fi, fj, fi >= 0 ? D[(size_t)fi * N + fj] : 0.0f);
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dS);
    return bad || hS[0] || hS[1];
}


// ---- mode 4 / 5: kind::f16 (bf16 operands) with A from tensor memory, packed two
// K-elements per 32-bit column, B from shared memory (K-major, 128-byte swizzle:
// 64 bf16 per row), accumulated onto a kind::tf32 product in the same
// accumulator: D = A32 * B32^T (tf32) + A16 * B16^T (bf16).
#include <cuda_bf16.h>
template <int CG>
__device__ __forceinline__ void mma_ts_bf16(unsigned d, unsigned a_tmem, unsigned long long b, unsigned idesc, unsigned acc) {
    if (CG == 1)
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int CG>
__global__ void __launch_bounds__(128) probe_mixed(const float *A32, const float *B32, const float *A16f, const float *B16f,
                                                   float *D, int *status) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    unsigned rank = 0;
    if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    constexpr int NB = N / CG;
    constexpr int B_ATOM = NB * 128;
    unsigned char *sB32 = smem;                            // K/32 atoms
    unsigned char *sB16 = smem + (K / 32) * B_ATOM;        // K/64 atoms
    const float *Br32 = B32 + (size_t)rank * NB * K, *Br16 = B16f + (size_t)rank * NB * K;
    for (int i = tid; i < NB * K; i += 128)
        *(float *)(sB32 + sw128_off(i / K, i % K, B_ATOM)) = Br32[i];
    for (int i = tid; i < NB * K; i += 128) {
        const int row = i / K, k = i % K;                  // bf16: 8 elements per 16-byte chunk, 64 per atom
        const int ka = k >> 6, c = (k & 63) >> 3;
        const unsigned off = ka * B_ATOM + (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4) + (k & 7) * 2;
        *(__nv_bfloat16 *)(sB16 + off) = __float2bfloat16(Br16[i]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)), "n"(512) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)), "n"(512) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base_s;
    {
        // A32: lane = row, column 128 + k.  A16: column 256 + k / 2 holds (k even: low half, k odd: high half)
        const float *a32 = A32 + ((size_t)rank * 128 + 32 * warp + lane) * K;
        const float *a16 = A16f + ((size_t)rank * 128 + 32 * warp + lane) * K;
        for (int k0 = 0; k0 < K; k0 += 32) {
            float v[32];
            for (int i = 0; i < 32; ++i) v[i] = a32[k0 + i];
            tmem_st32(tmem + ((unsigned)(32 * warp) << 16) + 128 + k0, v);
        }
        for (int k0 = 0; k0 < K; k0 += 64) {
            float v[32];
            for (int i = 0; i < 32; ++i) {
                __nv_bfloat162 p2 = __floats2bfloat162_rn(a16[k0 + 2 * i], a16[k0 + 2 * i + 1]);
                v[i] = __uint_as_float(*reinterpret_cast<unsigned *>(&p2));
            }
            tmem_st32(tmem + ((unsigned)(32 * warp) << 16) + 256 + k0 / 2, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (tid == 0 && rank == 0) {
        const unsigned mn = ((unsigned)(N >> 3) << 17) | ((unsigned)((128 * CG) >> 4) << 24);
        const unsigned idesc32 = (1u << 4) | (2u << 7) | (2u << 10) | mn;
        const unsigned idesc16 = (1u << 4) | (1u << 7) | (1u << 10) | mn;      // bf16 x bf16 -> f32
        for (int k = 0; k < K / 8; ++k)
            mma_ts<CG>(tmem, tmem + 128 + 8 * k, sw128_desc(smem_u32(sB32) + (k >> 2) * B_ATOM + (k & 3) * 32), idesc32, k > 0);
        for (int k = 0; k < K / 16; ++k)
            mma_ts_bf16<CG>(tmem, tmem + 256 + 8 * k, sw128_desc(smem_u32(sB16) + (k >> 2) * B_ATOM + (k & 3) * 32), idesc16, 1u);
        if (CG == 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((unsigned short)3) : "memory");
    }
    const bool ok = mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (!ok) {
        if (tid == 0) status[rank] = 1;
    } else {
        float v[32];
        tmem_ld32(tmem + ((unsigned)(32 * warp) << 16), v);
        for (int j = 0; j < N; ++j) D[((size_t)rank * 128 + 32 * warp + lane) * N + j] = v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (warp == 0) {
        if (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
    }
}

static float bf16_round(float x) { return __bfloat162float(__float2bfloat16(x)); }

template <int CG>
static int run_mixed(const char *name) {
    const int M = 128 * CG;
    std::vector<float> A32((size_t)M * K), B32((size_t)N * K), A16((size_t)M * K), B16((size_t)N * K), D((size_t)M * N, -1.0f);
    srand(4321);
    for (auto &x : A32) x = tf32_trunc((float)rand() / RAND_MAX + 0.01f);
    for (auto &x : B32) x = tf32_trunc((float)rand() / RAND_MAX - 0.3f);
    for (auto &x : A16) x = bf16_round((float)rand() / RAND_MAX - 0.5f);
    for (auto &x : B16) x = bf16_round((float)rand() / RAND_MAX + 0.2f);
    float *d[5]; int *dS, hS[2] = {0, 0};
    std::vector<float> *h[4] = {&A32, &B32, &A16, &B16};
    for (int i = 0; i < 4; ++i) { CK(cudaMalloc(&d[i], h[i]->size() * 4)); CK(cudaMemcpy(d[i], h[i]->data(), h[i]->size() * 4, cudaMemcpyHostToDevice)); }
    CK(cudaMalloc(&d[4], D.size() * 4)); CK(cudaMemcpy(d[4], D.data(), D.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dS, 8)); CK(cudaMemset(dS, 0, 8));
    const size_t smem = (K / 32) * (N / CG * 128) + (K / 64) * (N / CG * 128);
    CK(cudaFuncSetAttribute(probe_mixed<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CG); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, probe_mixed<CG>, (const float *)d[0], (const float *)d[1], (const float *)d[2], (const float *)d[3], d[4], dS));
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: kernel failed: %s\n", name, cudaGetErrorString(e)); return 2; }
    CK(cudaMemcpy(D.data(), d[4], D.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hS, dS, 8, cudaMemcpyDeviceToHost));
    double worst = 0.0; int bad = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            double ref = 0.0;
            for (int k = 0; k < K; ++k)
                ref += (double)A32[(size_t)i * K + k] * B32[(size_t)j * K + k] + (double)A16[(size_t)i * K + k] * B16[(size_t)j * K + k];
            const double err = fabs(ref - D[(size_t)i * N + j]) / (fabs(ref) + 1.0);
            if (err > worst) worst = err;
            if (err > 1e-4) ++bad;
        }
    printf("%s: timeout flags %d %d, worst rel err %.3e, bad %d of %d\n", name, hS[0], hS[1], worst, bad, M * N);
    return bad || hS[0] || hS[1];
}

// ---- MMA issue-rate benchmark: REP back-to-back tcgen05.mma (kind::tf32, K = 8)
// of shape (128 CG) x NN, A from shared memory (SS) or tensor memory (TS);
// cycles per MMA from clock64 around issue + commit + wait.
template <int CG, bool ATMEM, int NN>
__global__ void __launch_bounds__(128) mma_rate(long long *cycles, int rep) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    unsigned rank = 0;
    if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    constexpr int NB = NN / CG;
    constexpr int A_ATOM = 128 * 128, B_ATOM = NB * 128;
    unsigned char *sA = smem, *sB = smem + 4 * A_ATOM;
    for (int i = tid; i < (4 * A_ATOM + 4 * B_ATOM) / 4; i += 128) ((float *)smem)[i] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)), "n"(512) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_s)), "n"(512) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const unsigned tmem = tmem_base_s;
    long long t0 = 0;
    if (tid == 0 && rank == 0) {
        const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(NN >> 3) << 17) |
                               ((unsigned)((128 * CG) >> 4) << 24);
        t0 = clock64();
        for (int r = 0; r < rep; ++r) {
            const int k = r & 15, ka = k >> 2, ks = k & 3;
            const unsigned long long bd = sw128_desc(smem_u32(sB) + ka * B_ATOM + ks * 32);
            if (ATMEM) mma_ts<CG>(tmem, tmem + 256 + 8 * k, bd, idesc, 1u);
            else mma_ss<CG>(tmem, sw128_desc(smem_u32(sA) + ka * A_ATOM + ks * 32), bd, idesc, 1u);
        }
        if (CG == 1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((unsigned short)3) : "memory");
    }
    mbar_wait(&bar, 0);
    if (tid == 0 && rank == 0) cycles[0] = clock64() - t0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (warp == 0) {
        if (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512) : "memory");
    }
}

template <int CG, bool ATMEM, int NN>
static void rate(const char *name) {
    long long *d, h = 0;
    CK(cudaMalloc(&d, 8));
    const size_t smem = 4 * 128 * 128 + 4 * (NN / CG) * 128;
    CK(cudaFuncSetAttribute(mma_rate<CG, ATMEM, NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CG); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    const int rep = 4096;
    for (int it = 0; it < 2; ++it) {
        CK(cudaLaunchKernelEx(&cfg, mma_rate<CG, ATMEM, NN>, d, rep));
        CK(cudaDeviceSynchronize());
    }
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    printf("rate %s N=%d: %.1f cycles per MMA (floor %d)\n", name, NN, (double)h / rep, 128 * NN / 256);
    cudaFree(d);
}

int main(int argc, char **argv) {
    const int mode = argc > 1 ? atoi(argv[1]) : -1;
    int rc = 0;
    if (mode < 0 || mode == 0) rc |= run<1, false>("mode0 cg1 SS");
    if (mode < 0 || mode == 1) rc |= run<1, true>("mode1 cg1 TS");
    if (mode < 0 || mode == 2) rc |= run<2, false>("mode2 cg2 SS");
    if (mode < 0 || mode == 3) rc |= run<2, true>("mode3 cg2 TS");
    if (mode < 0 || mode == 4) rc |= run_mixed<1>("mode4 cg1 tf32 TS + bf16 TS, one accumulator");
    if (mode < 0 || mode == 5) rc |= run_mixed<2>("mode5 cg2 tf32 TS + bf16 TS, one accumulator");
    if (mode == 9) {
        rate<1, false, 32>("cg1 SS"); rate<1, false, 64>("cg1 SS"); rate<1, false, 128>("cg1 SS"); rate<1, false, 256>("cg1 SS");
        rate<1, true, 32>("cg1 TS"); rate<1, true, 64>("cg1 TS"); rate<1, true, 128>("cg1 TS"); rate<1, true, 256>("cg1 TS");
        rate<2, false, 32>("cg2 SS"); rate<2, false, 64>("cg2 SS"); rate<2, false, 128>("cg2 SS"); rate<2, false, 256>("cg2 SS");
        rate<2, true, 32>("cg2 TS"); rate<2, true, 64>("cg2 TS"); rate<2, true, 128>("cg2 TS"); rate<2, true, 256>("cg2 TS");
    }
    return rc;
}
