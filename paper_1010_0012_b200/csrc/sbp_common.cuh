// Shared device helpers for the grid BP kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sbp.h"

#define SBP_FULL_MASK 0xffffffffu

namespace sbp {

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
