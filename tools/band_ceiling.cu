// Practical ceiling of the band's instruction streams on B200 (sm_100a):
// the exact per-lane band loops of band_message (packed FFMA2 for
// sum-product; FADD2 + FMNMX3 for max-sum, two taps per FMNMX3) on register-
// resident h, no memory traffic, 4 warps per scheduler.  Reports algorithmic
// operations per second (2 per band candidate, as the roofline counts them)
// and per SM clock, so kernel fractions can be read against what the
// instruction stream itself can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -o tools/band_ceiling tools/band_ceiling.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_1010_0012_b200/csrc/sbp_common.cuh"

using namespace sbp;

struct WP { float2 wp[4][2 * 32 + 4]; };   // 4 tables: a per-repetition table keeps
                                            // the weights out of registers, as in the kernels

__device__ __forceinline__ float fmax3d(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// one message's band for a lane: taps t in [-R, VL + R), own h from registers,
// taps from a 16-register window (no shuffles or shared memory: the ceiling
// of the arithmetic alone)
template <int DOM, int VL, int R>
__global__ void __launch_bounds__(512, 1) k_band(const __grid_constant__ WP p, float *out,
                                                  unsigned long long *cyc, int reps) {
    float h[16];
    for (int i = 0; i < 16; ++i) h[i] = threadIdx.x * 1e-3f + i * 0.01f;
    float o[VL];
    for (int i = 0; i < VL; ++i) o[i] = 0.0f;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < reps; ++it) {
        const float2 *wp = p.wp[it & 3];
        if (DOM == 0) {
#pragma unroll
            for (int t = -R; t < VL + R; ++t)
#pragma unroll
                for (int i = 0; i < VL; i += 2) {
                    const int d = t - i;
                    if (d < -R || d > R + 1) continue;
                    fma2(o[i], o[i + 1], wp[d + R + 1], h[(t + R) & 15]);
                }
        } else {
#pragma unroll
            for (int t = -R; t < VL + R; t += 2)
#pragma unroll
                for (int i = 0; i < VL; i += 2) {
                    const int d0 = t - i, d1 = t + 1 - i;
                    const bool in0 = d0 >= -R && d0 <= R + 1, in1 = d1 >= -R && d1 <= R + 1;
                    float a0, a1, b0, b1;
                    if (in0) add2(a0, a1, wp[d0 + R + 1].x, wp[d0 + R + 1].y, h[(t + R) & 15], h[(t + R) & 15]);
                    if (in1) add2(b0, b1, wp[d1 + R + 1].x, wp[d1 + R + 1].y, h[(t + 1 + R) & 15], h[(t + 1 + R) & 15]);
                    if (in0 && in1) {
                        o[i] = fmax3d(o[i], a0, b0);
                        o[i + 1] = fmax3d(o[i + 1], a1, b1);
                    } else if (in0) {
                        o[i] = fmaxf(o[i], a0);
                        o[i + 1] = fmaxf(o[i + 1], a1);
                    } else if (in1) {
                        o[i] = fmaxf(o[i], b0);
                        o[i + 1] = fmaxf(o[i + 1], b1);
                    }
                }
        }
        // new h each repetition (keeps the loop from being hoisted)
#pragma unroll
        for (int i = 0; i < 16; i += 4) h[i] = o[i % VL];
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < VL; ++i) s += o[i];
    if (s == 1.5f) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename K>
void run(const char *name, K k, int VL, int R, WP &p, float *o, unsigned long long *cyc, int sms) {
    const int reps = 64;
    k<<<sms, 512>>>(p, o, cyc, reps);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<sms, 512>>>(p, o, cyc, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[1024];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += h[i];
    mean /= sms;
    // algorithmic candidates per lane per message: VL labels x (2R + 1) taps
    const double cand = (double)VL * (2 * R + 1);
    const double ops = 2.0 * cand * reps * 512.0 * sms;
    printf("{\"test\": \"%s\", \"VL\": %d, \"R\": %d, \"tops\": %.2f, \"ops_per_clk_per_sm\": %.1f, "
           "\"sm_clk_ghz\": %.3f, \"err\": \"%s\"}\n",
           name, VL, R, ops / ms / 1e9, 2.0 * cand * reps * 512.0 / mean, mean / (ms * 1e6),
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    WP p;
    for (int q = 0; q < 4; ++q)
        for (int k = 0; k < 2 * 32 + 4; ++k) p.wp[q][k] = make_float2(0.5f - k * 1e-3f, 0.25f + q * 1e-3f);
    float *o;
    unsigned long long *cyc;
    cudaMalloc(&o, 4);
    cudaMalloc(&cyc, 8 * 1024);
    run("band_sum", k_band<0, 16, 32>, 16, 32, p, o, cyc, sms);
    run("band_sum", k_band<0, 8, 32>, 8, 32, p, o, cyc, sms);
    run("band_sum", k_band<0, 8, 16>, 8, 16, p, o, cyc, sms);
    run("band_max", k_band<1, 8, 32>, 8, 32, p, o, cyc, sms);
    run("band_max", k_band<1, 8, 16>, 8, 16, p, o, cyc, sms);
    return 0;
}
