// Issue / pipe throughput of the instruction forms the band kernels use, on
// B200 (sm_100a), in warp instructions per SM clock (clock64 inside the
// kernel, so the number does not depend on the power-capped SM clock).
// Every thread runs CH independent chains; blocks of 1024 threads, one per SM
// (8 warps per scheduler).  Operands that the kernels take from the
// constant bank (band weights) come from kernel parameters here too.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes tools/pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
#define IT 2048

struct W2 { unsigned long long w[16]; float s[16]; };

__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r;
}
__device__ __forceinline__ float lo(unsigned long long v) {
    float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b;
}

// per test: instructions per iteration per chain (for the counts)
#define KERNEL(NAME, NI, INIT, BODY, FIN)                                          \
__global__ void __launch_bounds__(1024, 1) NAME(const __grid_constant__ W2 p, float *out, \
                                                unsigned long long *cyc) {         \
    INIT                                                                           \
    __syncthreads();                                                               \
    long long t0 = clock64();                                                      \
    _Pragma("unroll 1") for (int it = 0; it < IT; ++it) { BODY }                 \
    __syncthreads();                                                               \
    long long t1 = clock64();                                                      \
    FIN                                                                            \
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;                               \
}

// FFMA2: acc pair += w pair (constant bank) * broadcast h  (the band's sum form)
KERNEL(k_ffma2_c, 1,
    unsigned long long a[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { a[c] = pk(threadIdx.x, c); h[c] = threadIdx.x * 1e-3f + c; },
#pragma unroll
    for (int c = 0; c < CH; ++c)
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[c]) : "l"(p.w[c]), "l"(pk(h[c], h[c])));,
    float s = 0; for (int c = 0; c < CH; ++c) s += lo(a[c]); if (s == 1.5f) out[0] = s;)

// FFMA2: all register operands
KERNEL(k_ffma2_r, 1,
    unsigned long long a[CH]; unsigned long long b[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { a[c] = pk(threadIdx.x, c); b[c] = pk(c, 1.f); h[c] = threadIdx.x * 1e-3f + c; },
#pragma unroll
    for (int c = 0; c < CH; ++c)
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[c]) : "l"(b[(c + 1) % CH]), "l"(pk(h[c], h[c])));,
    float s = 0; for (int c = 0; c < CH; ++c) s += lo(a[c]) + lo(b[c]); if (s == 1.5f) out[0] = s;)

// scalar FFMA with a constant-bank weight
KERNEL(k_ffma_c, 1,
    float a[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { a[c] = threadIdx.x; h[c] = threadIdx.x * 1e-3f + c; },
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(a[c]) : "f"(p.s[c]), "f"(h[c]));,
    float s = 0; for (int c = 0; c < CH; ++c) s += a[c]; if (s == 1.5f) out[0] = s;)

// scalar FFMA, all registers
KERNEL(k_ffma_r, 1,
    float a[CH]; float h[CH]; float w[CH];
    for (int c = 0; c < CH; ++c) { a[c] = threadIdx.x; h[c] = threadIdx.x * 1e-3f + c; w[c] = c * 0.5f + threadIdx.y; },
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(a[c]) : "f"(w[c]), "f"(h[c]));,
    float s = 0; for (int c = 0; c < CH; ++c) s += a[c] + w[c]; if (s == 1.5f) out[0] = s;)

// FADD2: candidate pair = w pair (constant bank) + broadcast h
KERNEL(k_fadd2_c, 1,
    unsigned long long a[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { a[c] = pk(threadIdx.x, c); h[c] = threadIdx.x * 1e-3f + c; },
#pragma unroll
    for (int c = 0; c < CH; ++c)
        asm volatile("add.rn.f32x2 %0, %1, %0;" : "+l"(a[c]) : "l"(p.w[c]));,
    float s = 0; for (int c = 0; c < CH; ++c) s += lo(a[c]); if (s == 1.5f) out[0] = s;)

// FMNMX3 (three-input max)
KERNEL(k_fmnmx3, 1,
    float a[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { a[c] = threadIdx.x; h[c] = threadIdx.x * 1e-3f + c; },
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[c]) : "f"(h[c]), "f"(h[(c + 1) % CH]));,
    float s = 0; for (int c = 0; c < CH; ++c) s += a[c]; if (s == 1.5f) out[0] = s;)

// FMNMX (two-input)
KERNEL(k_fmnmx, 1,
    float a[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { a[c] = threadIdx.x; h[c] = threadIdx.x * 1e-3f + c; },
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[c]) : "f"(h[c]));,
    float s = 0; for (int c = 0; c < CH; ++c) s += a[c]; if (s == 1.5f) out[0] = s;)

// FADD2 + FMNMX3 1:1 (the max-sum band: a candidate pair, folded into an output)
KERNEL(k_maxband, 2,
    float o[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { o[c] = threadIdx.x; h[c] = threadIdx.x * 1e-3f + c; },
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        unsigned long long x;
        asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(x) : "l"(p.w[c]), "l"(pk(h[c], h[c])));
        float x0; float x1; asm("mov.b64 {%0,%1}, %2;" : "=f"(x0), "=f"(x1) : "l"(x));
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(o[c]) : "f"(x0), "f"(x1));
        h[c] = o[(c + 5) % CH];
    },
    float s = 0; for (int c = 0; c < CH; ++c) s += o[c]; if (s == 1.5f) out[0] = s;)

// FFMA2 + FSEL 1:1 (band FMAs with an alu-pipe select in between)
KERNEL(k_ffma2_sel, 2,
    unsigned long long a[CH]; float h[CH]; float q[CH];
    for (int c = 0; c < CH; ++c) { a[c] = pk(threadIdx.x, c); h[c] = threadIdx.x * 1e-3f + c; q[c] = c; },
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[c]) : "l"(p.w[c]), "l"(pk(h[c], h[c])));
        asm volatile("{.reg .pred pp; setp.gt.u32 pp, %2, 5; selp.f32 %0, %0, %1, pp;}" : "+f"(q[c]) : "f"(h[c]), "r"(threadIdx.x + c));
    },
    float s = 0; for (int c = 0; c < CH; ++c) s += lo(a[c]) + q[c]; if (s == 1.5f) out[0] = s;)

// SHFL
KERNEL(k_shfl, 1,
    float a[CH];
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x * 1e-3f + c;,
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = __shfl_down_sync(0xffffffffu, a[c], 1 + (c & 3), 16);,
    float s = 0; for (int c = 0; c < CH; ++c) s += a[c]; if (s == 1.5f) out[0] = s;)

// LDS.128 (shared-memory band taps)
KERNEL(k_lds128, 1,
    __shared__ float4 sm[1024 * 2]; float4 a[CH];
    sm[threadIdx.x] = make_float4(threadIdx.x, 1, 2, 3); sm[threadIdx.x + 1024] = sm[threadIdx.x];
    for (int c = 0; c < CH; ++c) a[c] = make_float4(0, 0, 0, 0);,
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        float4 v; int idx = (threadIdx.x + c * 33 + (int)a[c].w) & 2047;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"((unsigned)__cvta_generic_to_shared(&sm[idx])));
        a[c].x += v.x; a[c].w = v.w * 0.f;
    },
    float s = 0; for (int c = 0; c < CH; ++c) s += a[c].x; if (s == 1.5f) out[0] = s;)


// Clean forms (sm_100 intrinsics): FFMA2 with a broadcast multiplicand that
// changes every iteration (the band: acc pair += w pair * h), and the
// max-sum band pair FADD2 (w pair + h) -> FMNMX3 fold, 1:1.
struct F2W { float2 w[16]; };
__global__ void __launch_bounds__(1024, 1) k_ffma2_clean(const __grid_constant__ F2W p, float *out,
                                                        unsigned long long *cyc) {
    float2 a[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { a[c] = make_float2(threadIdx.x, c); h[c] = threadIdx.x * 1e-3f + c; }
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __ffma2_rn(p.w[c], make_float2(h[c], h[c]), a[c]);
#pragma unroll
        for (int c = 0; c < CH; ++c) h[c] = a[(c + 1) % CH].x;
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0; for (int c = 0; c < CH; ++c) s += a[c].x + a[c].y; if (s == 1.5f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void __launch_bounds__(1024, 1) k_maxband_clean(const __grid_constant__ F2W p, float *out,
                                                          unsigned long long *cyc) {
    float o[CH]; float h[CH];
    for (int c = 0; c < CH; ++c) { o[c] = threadIdx.x; h[c] = threadIdx.x * 1e-3f + c; }
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < IT; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const float2 x = __fadd2_rn(p.w[c], make_float2(h[c], h[c]));
            float r; asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(o[c]), "f"(x.x), "f"(x.y));
            o[c] = r;
        }
#pragma unroll
        for (int c = 0; c < CH; ++c) h[c] = o[(c + 3) % CH] * 0.5f;
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0; for (int c = 0; c < CH; ++c) s += o[c]; if (s == 1.5f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename P, typename K>
void run2(const char *name, K k, P &p, float *o, unsigned long long *cyc, int sms) {
    k<<<sms, 1024>>>(p, o, cyc);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<sms, 1024>>>(p, o, cyc);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[1024]; cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double mean = 0; for (int i = 0; i < sms; ++i) mean += h[i]; mean /= sms;
    printf("{\"test\": \"%s\", \"sm_clk_per_warp_iter\": %.4f, \"sm_clk_ghz\": %.3f, \"err\": \"%s\"}\n",
           name, mean / (32.0 * IT), mean / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
}

template <typename K>
void run(const char *name, K k, int ni, W2 &p, float *o, unsigned long long *cyc, int sms) {
    k<<<sms, 1024>>>(p, o, cyc);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<sms, 1024>>>(p, o, cyc);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[1024]; cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double mean = 0; for (int i = 0; i < sms; ++i) mean += h[i]; mean /= sms;
    // 32 warps per SM each run IT loop iterations: SM clocks per warp-iteration
    printf("{\"test\": \"%s\", \"sm_clk_per_warp_iter\": %.4f, "
           "\"sm_clk_ghz\": %.3f, \"err\": \"%s\"}\n",
           name, mean / (32.0 * IT), mean / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    W2 p; for (int i = 0; i < 16; ++i) { float a = 0.5f + i, b = 0.25f - i; memcpy(&p.w[i], &a, 4); memcpy((char *)&p.w[i] + 4, &b, 4); p.s[i] = 0.99f; }
    float *o; unsigned long long *cyc; cudaMalloc(&o, 4); cudaMalloc(&cyc, 8 * 1024);
    run("ffma2_constw", k_ffma2_c, 1, p, o, cyc, sms);
    run("ffma2_regs", k_ffma2_r, 1, p, o, cyc, sms);
    run("ffma_constw", k_ffma_c, 1, p, o, cyc, sms);
    run("ffma_regs", k_ffma_r, 1, p, o, cyc, sms);
    run("fadd2_constw", k_fadd2_c, 1, p, o, cyc, sms);
    run("fmnmx3", k_fmnmx3, 1, p, o, cyc, sms);
    run("fmnmx", k_fmnmx, 1, p, o, cyc, sms);
    run("fadd2+fmnmx3(maxband)", k_maxband, 2, p, o, cyc, sms);
    run("ffma2+fsel", k_ffma2_sel, 2, p, o, cyc, sms);
    run("shfl", k_shfl, 1, p, o, cyc, sms);
    run("lds128", k_lds128, 1, p, o, cyc, sms);
    F2W q; for (int i = 0; i < 16; ++i) q.w[i] = make_float2(0.5f + i * 1e-3f, 0.25f - i * 1e-3f);
    run2("ffma2_clean", k_ffma2_clean, q, o, cyc, sms);
    run2("maxband_clean", k_maxband_clean, q, o, cyc, sms);
    return 0;
}
