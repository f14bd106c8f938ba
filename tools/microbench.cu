// Pipe-throughput microbenchmarks on B200 (sm_100a): FP32 FFMA (the FP32
// roofline denominator, which MEASURED_PEAKS.json does not carry), FP64
// add/max, f32<->f64 conversions and warp shuffles.  Each thread runs
// independent dependency chains; throughput = ops / kernel time.
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

__global__ void k_ffma(float *out, float a, float b) {
    float v[CHAINS];
    for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) v[c] = fmaf(v[c], a, b);
    float s = 0; for (int c = 0; c < CHAINS; ++c) s += v[c];
    if (s == 1234.5f) out[0] = s;
}
__global__ void k_dadd(double *out, double a) {
    double v[CHAINS];
    for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) v[c] = v[c] + a;
    double s = 0; for (int c = 0; c < CHAINS; ++c) s += v[c];
    if (s == 1234.5) out[0] = s;
}
__global__ void k_dmax(double *out, double a) {
    double v[CHAINS];
    for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) v[c] = fmax(v[c], a + c);
    double s = 0; for (int c = 0; c < CHAINS; ++c) s += v[c];
    if (s == 1234.5) out[0] = s;
}
__global__ void k_cvt(float *out, float a) {
    float v[CHAINS];
    for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            double d = (double)v[c];          // F2F.F64.F32
            v[c] = (float)(d * 1.0000001);    // DMUL + F2F.F32.F64
        }
    float s = 0; for (int c = 0; c < CHAINS; ++c) s += v[c];
    if (s == 1234.5f) out[0] = s;
}
__global__ void k_fmax(float *out, float a) {
    float v[CHAINS];
    for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) v[c] = fmaxf(v[c] + a, v[(c + 1) % CHAINS]);
    float s = 0; for (int c = 0; c < CHAINS; ++c) s += v[c];
    if (s == 1234.5f) out[0] = s;
}
__global__ void k_shfl(float *out, float a) {
    float v[CHAINS];
    for (int c = 0; c < CHAINS; ++c) v[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) v[c] = __shfl_down_sync(0xffffffffu, v[c], 1 + (c & 3), 16);
    float s = 0; for (int c = 0; c < CHAINS; ++c) s += v[c];
    if (s == 1234.5f) out[0] = s;
}

template <typename F>
float timeit(F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    const double ops = (double)blocks * threads * ITERS * CHAINS;
    float *fo; double *dout; cudaMalloc(&fo, 4); cudaMalloc(&dout, 8);
    float t;
    t = timeit([&] { k_ffma<<<blocks, threads>>>(fo, 1.0001f, 0.5f); });
    printf("{\"op\": \"ffma\", \"tflops\": %.2f}\n", 2 * ops / t / 1e9);
    t = timeit([&] { k_dadd<<<blocks, threads>>>(dout, 1.0); });
    printf("{\"op\": \"dadd\", \"tops\": %.2f, \"per_clk_per_sm_at_1.9GHz\": %.1f}\n", ops / t / 1e9, ops / t * 1e3 / sms / 1.9e9);
    t = timeit([&] { k_dmax<<<blocks, threads>>>(dout, 1.0); });
    printf("{\"op\": \"dadd+dmax\", \"tops\": %.2f}\n", 2 * ops / t / 1e9);
    t = timeit([&] { k_cvt<<<blocks, threads>>>(fo, 1.0f); });
    printf("{\"op\": \"cvt f32->f64 + dmul + cvt f64->f32\", \"chains_per_s_T\": %.2f, \"per_clk_per_sm\": %.1f}\n", ops / t / 1e9, ops / t * 1e3 / sms / 1.9e9);
    t = timeit([&] { k_fmax<<<blocks, threads>>>(fo, 1.0f); });
    printf("{\"op\": \"fadd+fmax\", \"tops\": %.2f}\n", 2 * ops / t / 1e9);
    t = timeit([&] { k_shfl<<<blocks, threads>>>(fo, 1.0f); });
    printf("{\"op\": \"shfl\", \"warp_instr_per_clk_per_sm_at_1.9GHz\": %.2f}\n", ops / 32 / t * 1e3 / sms / 1.9e9);
    return 0;
}
