// Shared device helpers for the grid BP kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sbp.h"

#define SBP_FULL_MASK 0xffffffffu

namespace sbp {

// Upper bound on the blocks of a persistent (grid-stride) launch: 0 = no cap
// beyond residency.  SBP_MAX_BLOCKS (read once, sbp_reload_config) changes the
// launch geometry for race checks (tests/test_gpu_guards.py).  Defined in capi.cu.
int launch_block_cap();

// Reference directed-edge id (bp.py:113-133 over the edge order of
// mrf.py:401-411): node-major, each node emits (n, n+1) then (n, n+W);
// undirected edge e yields 2e for a->b and 2e+1 for b->a.
__device__ __forceinline__ long long edge_base(long long r, long long c, long long H,
                                               long long W) {
    return r * (2 * W - 1) + (r < H - 1 ? 2 * c : c);
}

// dir: 0 send right (L->R pass), 1 send left, 2 send down (T->B), 3 send up.
__device__ __forceinline__ long long directed_edge_id(long long H, long long W, long long r,
                                                      long long c, int dir) {
    switch (dir) {
    case 0: return 2 * edge_base(r, c, H, W);
    case 1: return 2 * edge_base(r, c - 1, H, W) + 1;
    case 2: return 2 * (edge_base(r, c, H, W) + (c + 1 < W ? 1 : 0));
    default: return 2 * (edge_base(r - 1, c, H, W) + (c + 1 < W ? 1 : 0)) + 1;
    }
}

__device__ __forceinline__ void report_failure(unsigned long long *err, int iteration,
                                               long long edge_id) {
    unsigned long long key = ((unsigned long long)iteration << 40) |
                             (unsigned long long)edge_id;
    atomicMin(err, key);
}

// Geometry of the four outgoing directions (numba_kernels.py:230-245):
// excluded incoming slot, slot written in the neighbour, orientation.
__host__ __device__ constexpr int dir_excl(int d) { return d == 0 ? 2 : d == 1 ? 1 : d == 2 ? 3 : 0; }
__host__ __device__ constexpr int dir_wslot(int d) { return d == 0 ? 1 : d == 1 ? 2 : d == 2 ? 0 : 3; }
__host__ __device__ constexpr int dir_orient(int d) { return (d == 0 || d == 2) ? 0 : 1; }

// Packed FP32 pairs (sm_100 FADD2 / FMUL2 / FFMA2).  Each half rounds exactly
// like the scalar instruction (IEEE round-to-nearest, no contraction), so a
// packed loop gives the same bits as the scalar one with half the issue slots.
__device__ __forceinline__ unsigned long long f2_pack(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}

__device__ __forceinline__ void f2_unpack(unsigned long long v, float &a, float &b) {
    asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}

#ifndef SBP_SCALAR_F32
// (r0, r1) = (a0 + b0, a1 + b1)
__device__ __forceinline__ void add2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a0, a1)), "l"(f2_pack(b0, b1)));
    f2_unpack(r, r0, r1);
}

// (r0, r1) = (a0 - b0, a1 - b1)
__device__ __forceinline__ void sub2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a0, a1)), "l"(f2_pack(b0, b1)));
    f2_unpack(r, r0, r1);
}

// (r0, r1) = (a0 * b0, a1 * b1)
__device__ __forceinline__ void mul2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_pack(a0, a1)), "l"(f2_pack(b0, b1)));
    f2_unpack(r, r0, r1);
}

// (o0, o1) = (fma(w.x, x, o0), fma(w.y, x, o1))
__device__ __forceinline__ void fma2(float &o0, float &o1, float2 w, float x) {
    unsigned long long r = f2_pack(o0, o1);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(f2_pack(w.x, w.y)), "l"(f2_pack(x, x)));
    f2_unpack(r, o0, o1);
}

// (o0, o1) = (fma(x0, w, o0), fma(x1, w, o1)): one weight for a label pair
__device__ __forceinline__ void fma2b(float &o0, float &o1, float x0, float x1, float w) {
    unsigned long long r = f2_pack(o0, o1);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(f2_pack(x0, x1)), "l"(f2_pack(w, w)));
    f2_unpack(r, o0, o1);
}
#else
// Scalar build (A/B comparisons only): the same roundings one lane at a time.
__device__ __forceinline__ void add2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    r0 = __fadd_rn(a0, b0); r1 = __fadd_rn(a1, b1);
}
__device__ __forceinline__ void sub2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    r0 = __fsub_rn(a0, b0); r1 = __fsub_rn(a1, b1);
}
__device__ __forceinline__ void mul2(float &r0, float &r1, float a0, float a1, float b0, float b1) {
    r0 = __fmul_rn(a0, b0); r1 = __fmul_rn(a1, b1);
}
__device__ __forceinline__ void fma2(float &o0, float &o1, float2 w, float x) {
    o0 = fmaf(w.x, x, o0); o1 = fmaf(w.y, x, o1);
}
__device__ __forceinline__ void fma2b(float &o0, float &o1, float x0, float x1, float w) {
    o0 = fmaf(x0, w, o0); o1 = fmaf(x1, w, o1);
}
#endif

// Knuth TwoSum on a pair: a + b = s + e exactly, per half (adds only).
__device__ __forceinline__ void two_sum2(float a0, float a1, float b0, float b1, float &s0,
                                         float &s1, float &e0, float &e1) {
    float bp0, bp1, t0, t1, u0, u1, v0, v1;
    add2(s0, s1, a0, a1, b0, b1);
    sub2(bp0, bp1, s0, s1, a0, a1);
    sub2(t0, t1, s0, s1, bp0, bp1);
    sub2(u0, u1, a0, a1, t0, t1);
    sub2(v0, v1, b0, b1, bp0, bp1);
    add2(e0, e1, u0, u1, v0, v1);
}

__device__ __forceinline__ float4 ldg_stream(const float4 *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void stg_stream(float4 *p, float4 v) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

}  // namespace sbp
