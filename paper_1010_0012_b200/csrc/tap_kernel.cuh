// Wide-band synchronous BP iteration with the band's taps exchanged through
// shared memory (sm_100a).
//
// Same arithmetic as band_iter_kernel (band_kernel.cuh): per node the
// exclusion vectors h_{i\j} in the reference order (numba_kernels.py:194-227),
// the fast update (Eq. 7 / Eq. 11, numba_kernels.py:44-54 / 77-90) and the
// reference normalisation (:248-271) -- every output accumulates the same
// terms in the same order, so results are bit-identical to the shuffle
// kernels.  What changes is how a lane gets the h values of the labels owned
// by its neighbouring lanes (the out-of-lane taps, R on each side):
//
//   shuffle kernels: one SHFL + one pad select per tap (2R of each per lane
//   and message; SHFL issues at 1 warp-instruction / clock / SM), and all
//   2R taps live in registers (138 registers at R = 32: 12 warps / SM);
//
//   here: every lane stores its VL labels of h into its node's row in shared
//   memory and streams the band window back in 4-tap chunks (LDS.128), right
//   where the FMAs / max-adds consume them.  The row carries R pad labels
//   (0 / -inf) on both sides, written once per launch, so no selects are
//   needed, and taps never occupy more than one 4-float chunk of registers.
//
// Rows use a sub-row layout (TapRow) so the 8 lanes of each LDS.128 /
// STS.128 phase read 8 consecutive 16-byte slots: conflict-free, and every
// access is a per-lane base pointer plus an immediate offset.
#pragma once

#include "band_kernel.cuh"

namespace sbp {

// Row of one node's h in shared memory: PADL pad labels, Ms labels, PADL pad
// labels, as 4-float chunks k.  Lane j owns chunks k = PADL/4 + S j + ...
// (S = VL/4 chunks per lane), so the 8 lanes of an LDS.128 / STS.128 phase
// touch chunks c, c + S, ..., c + 7 S.  The row is stored as S sub-rows by
// k mod S (chunk k at (k / S) + (k mod S) * NCH/S): those 8 chunks are then 8
// CONSECUTIVE 16-byte slots -- 8 distinct bank groups, conflict-free -- and,
// because k mod S and the k / S offset depend only on the compile-time tap
// offset, every access is the lane's base pointer plus an immediate.
template <int MS, int VL>
struct TapRow {
    static constexpr int PADL = 32;                  // >= SBP_MAX_R, multiple of 32
    static constexpr int L = MS + 2 * PADL;          // floats
    static constexpr int PHYS = L;
    static constexpr int S = VL / 4;                 // lane stride in chunks
    static constexpr int NCH = L / 4;
    static constexpr int QS = NCH / S;               // chunks per sub-row
    static_assert(NCH % S == 0 && (PADL / 4) % S == 0, "sub-row layout");
    // physical float offset of logical float y (row initialisation)
    static __device__ __forceinline__ int phys(int y) {
        const int k = y >> 2;
        return 4 * ((k / S) + (k % S) * QS) + (y & 3);
    }
    // float offset, from the lane's base (row + 4 j), of the chunk holding the
    // lane's labels x0 + t .. x0 + t + 3 (t a multiple of 4, |t| <= PADL)
    static __device__ __forceinline__ constexpr int off(int t) {
        return 4 * ((PADL / 4 + t / 4) / S + ((PADL / 4 + t / 4) % S) * QS);
    }
};

__device__ __forceinline__ float4 lds128(const float *p) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}

__device__ __forceinline__ void sts128(float *p, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "f"(a), "f"(b),
                 "f"(c), "f"(d)
                 : "memory");
}

// The message of one directed edge from its exclusion vector h, taps from the
// node's shared-memory row.  Identical arithmetic and order to band_message.
template <int DOM, int VL, int LP, int R, int O>
__device__ __forceinline__ bool tap_message(const BandArgs &a, const float (&h)[VL], int x0,
                                            float *row, float (&out)[VL]) {
    static_assert(R % 4 == 0 && VL % 4 == 0, "4-tap chunks");
    using Row = TapRow<VL * LP, VL>;
    // publish h: the previous message's reads of the row are complete
    __syncwarp();
#pragma unroll
    for (int i = 0; i < VL; i += 4)
        sts128(row + 4 * (x0 / VL) + Row::off(i), h[i], h[i + 1], h[i + 2], h[i + 3]);
    if (DOM == SBP_SUM) {
        const float s = lanes_sum<LP>(vsum(h));
        const float base = a.floor_term ? a.fbar[O] * s : 0.0f;
#pragma unroll
        for (int i = 0; i < VL; ++i) out[i] = base;
    } else {
        float mx = fmaxf(h[0], h[1]);
#pragma unroll
        for (int i = 2; i < VL; i += 2) mx = fmax3(mx, h[i], h[i + 1]);
        mx = lanes_max<LP>(mx);
        const float base = a.floor_term ? a.fbar[O] + mx : -__builtin_huge_valf();
#pragma unroll
        for (int i = 0; i < VL; ++i) out[i] = base;
    }
    __syncwarp();
    // Band in ascending x_i, 4 taps at a time: term (x_i = x0 + t) reaches
    // out[i] at d = t - i; label pairs take the weight pair (w(d), w(d-1)).
#pragma unroll
    for (int tc = -R; tc < VL + R; tc += 4) {
        float hv[4];
        if (tc >= 0 && tc < VL) {
            hv[0] = h[tc]; hv[1] = h[tc + 1]; hv[2] = h[tc + 2]; hv[3] = h[tc + 3];
        } else {
            const float4 v = lds128(row + 4 * (x0 / VL) + Row::off(tc));
            hv[0] = v.x; hv[1] = v.y; hv[2] = v.z; hv[3] = v.w;
        }
        if (DOM == SBP_SUM) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = tc + u;
#pragma unroll
                for (int i = 0; i < VL; i += 2) {
                    const int d = t - i;
                    if (d < -R || d > R + 1) continue;
                    fma2(out[i], out[i + 1], a.wp[O][d + R + 1], hv[u]);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
                const int t = tc + u;
#pragma unroll
                for (int i = 0; i < VL; i += 2) {
                    const int d0 = t - i, d1 = t + 1 - i;
                    const bool in0 = d0 >= -R && d0 <= R + 1;
                    const bool in1 = d1 >= -R && d1 <= R + 1;
                    float a0, a1, b0, b1;
                    if (in0) add2(a0, a1, a.wp[O][d0 + R + 1].x, a.wp[O][d0 + R + 1].y, hv[u], hv[u]);
                    if (in1) add2(b0, b1, a.wp[O][d1 + R + 1].x, a.wp[O][d1 + R + 1].y, hv[u + 1], hv[u + 1]);
                    if (in0 && in1) {
                        out[i] = fmax3(out[i], a0, b0);
                        out[i + 1] = fmax3(out[i + 1], a1, b1);
                    } else if (in0) {
                        out[i] = fmaxf(out[i], a0);
                        out[i + 1] = fmaxf(out[i + 1], a1);
                    } else if (in1) {
                        out[i] = fmaxf(out[i], b0);
                        out[i + 1] = fmaxf(out[i + 1], b1);
                    }
                }
            }
        }
    }
    bool ok;
    if (DOM == SBP_SUM) {
        if (a.M < a.Ms) {
#pragma unroll
            for (int i = 0; i < VL; ++i)
                if (x0 + i >= a.M) out[i] = 0.0f;
        }
        const float s = lanes_sum<LP>(vsum(out));
        ok = (s > 0.0f) && !isinf(s);
        const float inv = __frcp_rn(s);
#pragma unroll
        for (int i = 0; i < VL; i += 2) mul2(out[i], out[i + 1], out[i], out[i + 1], inv, inv);
    } else {
        if (a.M < a.Ms) {
#pragma unroll
            for (int i = 0; i < VL; ++i)
                if (x0 + i >= a.M) out[i] = -__builtin_huge_valf();
        }
        float mx = fmaxf(out[0], out[1]);
#pragma unroll
        for (int i = 2; i < VL; i += 2) mx = fmax3(mx, out[i], out[i + 1]);
        mx = lanes_max<LP>(mx);
        ok = isfinite(mx);
#pragma unroll
        for (int i = 0; i < VL; i += 2) sub2(out[i], out[i + 1], out[i], out[i + 1], mx, mx);
    }
    return ok;
}

template <int DOM, int VL, int LP, int R, int O>
__device__ __forceinline__ void tap_emit(const BandArgs &a, const IterCtx &it, const float (&h)[VL],
                                         int DIR, int j, int x0, float *row, bool active,
                                         long long node_l, long long r, int c) {
    float out[VL];
    const bool ok = tap_message<DOM, VL, LP, R, O>(a, h, x0, row, out);
    if (!active) return;
    const long long W = a.W;
    const long long step = DIR == 0 ? 1 : DIR == 1 ? -1 : DIR == 2 ? W : -W;
    const long long dir_off = dir_wslot(DIR) * a.slot_stride + step * a.Ms;
    float *dst = it.msgs_out + (node_l * a.Ms + x0) + dir_off;
    if (a.delta)
        *it.dmax = fmaxf(*it.dmax, message_delta<DOM, VL>(out, it.msgs_in + (node_l * a.Ms + x0) + dir_off,
                                                         it.first, x0, a.M));
    Vec8Loader<VL>::store(dst, out);
    if (!ok && j == 0) report_failure(a.err, it.iteration, directed_edge_id(a.H, W, r, c, DIR));
}

// The four messages of one node (unrolled directions or a runtime loop over
// one band copy for symmetric potentials), the reference exclusion order and
// the error-free max-sum h of band_group_body / band_group_body_rolled.
template <int DOM, int VL, int LP, int R, bool ROLLED>
__device__ __forceinline__ void tap_group_body(const BandArgs &a, const IterCtx &it, const float (&g)[VL],
                                               const float (&m0)[VL], const float (&m1)[VL],
                                               const float (&m2)[VL], const float (&m3)[VL], int j,
                                               int x0, float *row, bool valid, long long node_l,
                                               long long r, int c) {
    const unsigned has = (c + 1 < a.W ? 1u : 0u) | (c > 0 ? 2u : 0u) |
                         (r + 1 < a.H ? 4u : 0u) | (r > 0 ? 8u : 0u);
    float pa[VL], pb[VL], ea[VL], eb[VL];
    if (DOM == SBP_SUM) {
        vmul(pa, g, m0);
        vmul(pb, pa, m1);
    } else {
        vtwo_sum(g, m0, pa, ea);
        vtwo_sum_from(pa, ea, m1, pb, eb);
    }
    auto one = [&](int dir) {
        const bool hd = (has >> dir) & 1u;
        if (!__any_sync(SBP_FULL_MASK, valid && hd)) return;
        float h[VL];
        if (DOM == SBP_SUM) {
            if (dir == 3) {
                vmul(h, g, m1);
                vmul(h, h, m2);
                vmul(h, h, m3);
            } else if (dir == 1) {
                vmul(h, pa, m2);
                vmul(h, h, m3);
            } else if (dir == 0) {
                vmul(h, pb, m3);
            } else {
                vmul(h, pb, m2);
            }
        } else {
            float s2[VL], e2[VL];
            if (dir == 3) {
                vtwo_sum(g, m1, s2, e2);
                vtwo_sum_acc(s2, m2, e2, e2);
                vtwo_sum_acc(s2, m3, e2, e2);
            } else if (dir == 1) {
                vtwo_sum_from(pa, ea, m2, s2, e2);
                vtwo_sum_acc(s2, m3, e2, e2);
            } else if (dir == 0) {
                vtwo_sum_from(pb, eb, m3, s2, e2);
            } else {
                vtwo_sum_from(pb, eb, m2, s2, e2);
            }
            shift_compensated<VL, LP>(s2, e2, h);
        }
        if (ROLLED) {
            tap_emit<DOM, VL, LP, R, 0>(a, it, h, dir, j, x0, row, valid && hd, node_l, r, c);
        } else if (dir == 0 || dir == 2) {
            tap_emit<DOM, VL, LP, R, 0>(a, it, h, dir, j, x0, row, valid && hd, node_l, r, c);
        } else {
            tap_emit<DOM, VL, LP, R, 1>(a, it, h, dir, j, x0, row, valid && hd, node_l, r, c);
        }
    };
    if constexpr (ROLLED) {
#pragma unroll 1
        for (int k = 0; k < 4; ++k) one((0x2013 >> (4 * k)) & 0xF);   // order 3, 1, 0, 2
    } else {
        one(3);
        one(1);
        one(0);
        one(2);
    }
}

constexpr int TAP_WARPS = 4;

// Per-warp shared memory: PPW node rows + (staged) NS stages of 5 input
// vectors for the warp's pixel group.
template <int VL, int LP, int NS>
struct TapSmem {
    static constexpr int PPW = 32 / LP;
    static constexpr int ROWF = TapRow<VL * LP, VL>::PHYS;
    static constexpr int ROWS_F = PPW * ROWF;                  // floats of the rows
    static constexpr int STAGE_F = NS * 5 * 32 * VL;           // floats of the input stages
    static constexpr int WARP_F = (ROWS_F + 31) / 32 * 32 + STAGE_F;
    static constexpr size_t bytes() { return (size_t)TAP_WARPS * WARP_F * sizeof(float); }
};

// Pad labels of a warp's rows: PADL floats on each side, the combining
// identity's absorbing value (0 for sums, -inf for maxima).  Written once.
template <int DOM, int VL, int LP>
__device__ __forceinline__ void tap_rows_init(float *rows) {
    using Row = TapRow<VL * LP, VL>;
    constexpr int PPW = 32 / LP;
    constexpr float PAD = DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    const int lane = threadIdx.x & 31;
    for (int k = lane; k < PPW * 2 * Row::PADL / 4; k += 32) {
        const int node = k / (2 * Row::PADL / 4), q = k % (2 * Row::PADL / 4);
        const int y = q < Row::PADL / 4 ? 4 * q : Row::PADL + VL * LP + 4 * (q - Row::PADL / 4);
        sts128(rows + node * Row::PHYS + Row::phys(y), PAD, PAD, PAD, PAD);
    }
    __syncwarp();
}

// NS = 0: register-loaded inputs (256-bit LDG); NS = 1 / 2: TMA-staged inputs
// (one / two stages of 1-D bulk copies per warp, as band_iter_staged_kernel).
// Resident blocks per SM.  VL = 16: 4 blocks (126-128 registers, no spills)
// instead of 3 (146 registers) -- slower cold (C4 2.49 vs 2.26 ms, C5 T=9 1.60
// vs 1.52) but faster where the benchmark and any workload longer than the
// power-cap response live: sustained at ~990 W C4 2.38 vs 2.48 ms per iteration
// (0.93 vs 0.89 of the copy peak), C5 T=9 1.57 vs 1.65 (0.94 vs 0.89;
// profiles/r02_ab_c4_tap_blocks.txt, r02_ab_t9_tap_blocks.txt).
#ifndef SBP_TAP16_BLOCKS
#define SBP_TAP16_BLOCKS(MS) 4
#endif
template <int DOM, int VL, int LP, int R, bool ROLLED, int NS>
__global__ void __launch_bounds__(32 * TAP_WARPS, (VL == 8 ? 4 : SBP_TAP16_BLOCKS(VL * LP)))
band_iter_tap_kernel(const __grid_constant__ BandArgs a) {
    using SM = TapSmem<VL, LP, NS>;
    constexpr int PPW = 32 / LP;
    constexpr int VEC = 32 * VL;
    float dmax = 0.0f;
    const IterCtx it = iter_of(a, &dmax);
    extern __shared__ __align__(128) float tap_smem[];
    __shared__ __align__(8) unsigned long long bars[TAP_WARPS][2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = lane % LP, q = lane / LP;
    const int x0 = j * VL;
    float *wbase = tap_smem + warp * SM::WARP_F;
    float *row = wbase + q * TapRow<VL * LP, VL>::PHYS;
    float *buf = wbase + (SM::ROWS_F + 31) / 32 * 32;
    tap_rows_init<DOM, VL, LP>(wbase);
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long ngroups = (npix + PPW - 1) / PPW;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;

    if constexpr (NS > 0) {
        if (lane == 0) {
            mbar_init(&bars[warp][0], 1);
            mbar_init(&bars[warp][1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const int nvec = a.first ? 1 : 5;
    auto issue = [&](long long gg, int st) {
        if (lane == 0) {
            const long long p0 = gg * PPW;
            const long long n = npix - p0 < PPW ? npix - p0 : PPW;
            const unsigned bytes = (unsigned)(n * a.Ms * 4);
            float *dst = buf + st * 5 * VEC;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bars[warp][st], bytes * nvec);
            bulk_g2s(dst, a.values + ((long long)(a.lr_begin - 1) * a.W + p0) * a.Ms, bytes,
                     &bars[warp][st]);
            if (!a.first)
                for (int k = 0; k < 4; ++k)
                    bulk_g2s(dst + (1 + k) * VEC,
                             a.msgs_in + k * a.slot_stride + ((long long)a.lr_begin * a.W + p0) * a.Ms,
                             bytes, &bars[warp][st]);
        }
    };
    unsigned phase = 0;
    int st = 0;
    if (NS > 0 && grp < ngroups) issue(grp, 0);
    for (; grp < ngroups; grp += nwarps) {
        if (NS == 2 && grp + nwarps < ngroups) issue(grp + nwarps, st ^ 1);
        long long p = grp * PPW + q;
        const bool valid = p < npix;
        if (!valid) p = npix - 1;
        const int lr = it.lr_begin + (int)(p / a.W);
        const int c = (int)(p % a.W);
        const long long r = (long long)a.r0 + lr - 1;
        const long long node_l = (long long)lr * a.W + c;
        float g[VL], m0[VL], m1[VL], m2[VL], m3[VL];
        if constexpr (NS == 0) {
            Vec8Loader<VL>::load(g, a.values + ((long long)(lr - 1) * a.W + c) * a.Ms + x0);
            if (!it.first) {
                const float *mi = it.msgs_in + node_l * a.Ms + x0;
                Vec8Loader<VL>::load(m0, mi);
                Vec8Loader<VL>::load(m1, mi + a.slot_stride);
                Vec8Loader<VL>::load(m2, mi + 2 * a.slot_stride);
                Vec8Loader<VL>::load(m3, mi + 3 * a.slot_stride);
            }
        } else {
            mbar_wait(&bars[warp][st], (phase >> st) & 1);
            phase ^= 1u << st;
            const float *src = buf + st * 5 * VEC + q * a.Ms + x0;
#pragma unroll
            for (int i = 0; i < VL; i += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(src + i);
                g[i] = v.x; g[i + 1] = v.y; g[i + 2] = v.z; g[i + 3] = v.w;
            }
            if (!it.first) {
                float *mm[4] = {m0, m1, m2, m3};
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int i = 0; i < VL; i += 4) {
                        const float4 v = *reinterpret_cast<const float4 *>(src + (1 + k) * VEC + i);
                        mm[k][i] = v.x; mm[k][i + 1] = v.y; mm[k][i + 2] = v.z; mm[k][i + 3] = v.w;
                    }
            }
            __syncwarp();   // every lane has read stage st before it is refilled
            if (NS == 1 && grp + nwarps < ngroups) issue(grp + nwarps, 0);
        }
        if (it.first) {
            // bp.py:587-601 without touching memory (see band_group)
            const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
            float *mm[4] = {m0, m1, m2, m3};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float real = DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M) : 0.0f;
#pragma unroll
                for (int i = 0; i < VL; ++i)
                    mm[k][i] = x0 + i < a.M ? real : (DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf());
            }
        }
        tap_group_body<DOM, VL, LP, R, ROLLED>(a, it, g, m0, m1, m2, m3, j, x0, row, valid, node_l,
                                               r, c);
        if (NS == 2) st ^= 1;
    }
    if (a.delta) flush_delta(a.delta, dmax);
}

template <int DOM, int VL, int LP, int R, bool ROLLED, int NS>
cudaError_t launch_band_tap(const BandArgs &a, cudaStream_t s) {
    constexpr int PPW = 32 / LP;
    using SM = TapSmem<VL, LP, NS>;
    const size_t smem = SM::bytes();
    static int resident = 0, sms = 0;
    if (!resident) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(band_iter_tap_kernel<DOM, VL, LP, R, ROLLED, NS>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &resident, band_iter_tap_kernel<DOM, VL, LP, R, ROLLED, NS>, 32 * TAP_WARPS, smem);
        if (resident < 1) resident = 1;
    }
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long warps = (npix + PPW - 1) / PPW;
    long long blocks = (warps + TAP_WARPS - 1) / TAP_WARPS;
    if (blocks <= 0) return cudaSuccess;
    const long long cap = (long long)sms * resident;
    if (blocks > cap) blocks = cap;
    if (launch_block_cap() > 0 && blocks > launch_block_cap()) blocks = launch_block_cap();
    band_iter_tap_kernel<DOM, VL, LP, R, ROLLED, NS><<<(unsigned)blocks, 32 * TAP_WARPS, smem, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// v2: register-light.  The four exclusion vectors of a node are formed once
// (reference order, prefix-shared, error-free for max-sum) straight into four
// shared-memory rows, so the input vectors die before the first band and no
// h state crosses the direction loop: ~60 registers instead of 125-140, i.e.
// 6-8 resident 4-warp blocks per SM instead of 3-4.  Each message then
// streams its whole window (own labels and taps) from its row.
// ---------------------------------------------------------------------------

// Sum (S) or max (H) of a lane's h over the node, as band_message forms it.
template <int DOM, int VL, int LP, bool RX = false>
__device__ __forceinline__ float node_reduce(const float (&h)[VL]) {
    if (DOM == SBP_SUM) return lanes_sum<LP>(vsum(h));
    float mx = fmaxf(h[0], h[1]);
#pragma unroll
    for (int i = 2; i < VL; i += 2) mx = fmax3(mx, h[i], h[i + 1]);
    return lanes_max<LP, RX>(mx);
}

// The v2 kernels reduce maxima with redux.sync (lanes_max) where it measured faster.
template <int DOM, int LP, int R>
constexpr bool tap2_redux() { return band_redux<DOM, LP, R>(); }

template <int DOM, int VL, int LP>
__device__ __forceinline__ void put_row(float *row, int x0, const float (&h)[VL]) {
    using Row = TapRow<VL * LP, VL>;
#pragma unroll
    for (int i = 0; i < VL; i += 4)
        sts128(row + 4 * (x0 / VL) + Row::off(i), h[i], h[i + 1], h[i + 2], h[i + 3]);
}

// One message from the node's row of direction `dir` (floor reduction `red`).
template <int DOM, int VL, int LP, int R, int O>
__device__ __forceinline__ bool tap2_message(const BandArgs &a, float red, int x0, const float *row,
                                             float (&out)[VL]) {
    using Row = TapRow<VL * LP, VL>;
    const float base = DOM == SBP_SUM ? (a.floor_term ? a.fbar[O] * red : 0.0f)
                                      : (a.floor_term ? a.fbar[O] + red : -__builtin_huge_valf());
#pragma unroll
    for (int i = 0; i < VL; ++i) out[i] = base;
#pragma unroll
    for (int tc = -R; tc < VL + R; tc += 4) {
        const float4 v = lds128(row + 4 * (x0 / VL) + Row::off(tc));
        const float hv[4] = {v.x, v.y, v.z, v.w};
        if (DOM == SBP_SUM) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int t = tc + u;
#pragma unroll
                for (int i = 0; i < VL; i += 2) {
                    const int d = t - i;
                    if (d < -R || d > R + 1) continue;
                    fma2(out[i], out[i + 1], a.wp[O][d + R + 1], hv[u]);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
                const int t = tc + u;
#pragma unroll
                for (int i = 0; i < VL; i += 2) {
                    const int d0 = t - i, d1 = t + 1 - i;
                    const bool in0 = d0 >= -R && d0 <= R + 1;
                    const bool in1 = d1 >= -R && d1 <= R + 1;
                    float a0, a1, b0, b1;
                    if (in0) add2(a0, a1, a.wp[O][d0 + R + 1].x, a.wp[O][d0 + R + 1].y, hv[u], hv[u]);
                    if (in1) add2(b0, b1, a.wp[O][d1 + R + 1].x, a.wp[O][d1 + R + 1].y, hv[u + 1], hv[u + 1]);
                    if (in0 && in1) {
                        out[i] = fmax3(out[i], a0, b0);
                        out[i + 1] = fmax3(out[i + 1], a1, b1);
                    } else if (in0) {
                        out[i] = fmaxf(out[i], a0);
                        out[i + 1] = fmaxf(out[i + 1], a1);
                    } else if (in1) {
                        out[i] = fmaxf(out[i], b0);
                        out[i + 1] = fmaxf(out[i + 1], b1);
                    }
                }
            }
        }
    }
    bool ok;
    if (DOM == SBP_SUM) {
        if (a.M < a.Ms) {
#pragma unroll
            for (int i = 0; i < VL; ++i)
                if (x0 + i >= a.M) out[i] = 0.0f;
        }
        const float s = lanes_sum<LP>(vsum(out));
        ok = (s > 0.0f) && !isinf(s);
        const float inv = __frcp_rn(s);
#pragma unroll
        for (int i = 0; i < VL; i += 2) mul2(out[i], out[i + 1], out[i], out[i + 1], inv, inv);
    } else {
        if (a.M < a.Ms) {
#pragma unroll
            for (int i = 0; i < VL; ++i)
                if (x0 + i >= a.M) out[i] = -__builtin_huge_valf();
        }
        float mx = fmaxf(out[0], out[1]);
#pragma unroll
        for (int i = 2; i < VL; i += 2) mx = fmax3(mx, out[i], out[i + 1]);
        mx = lanes_max<LP, tap2_redux<DOM, LP, R>()>(mx);
        ok = isfinite(mx);
#pragma unroll
        for (int i = 0; i < VL; i += 2) sub2(out[i], out[i + 1], out[i], out[i + 1], mx, mx);
    }
    return ok;
}

template <int DOM, int VL, int LP, int R, int O>
__device__ __forceinline__ void tap2_emit(const BandArgs &a, const IterCtx &it, float red,
                                          const float *row, int DIR, int j, int x0, bool active,
                                          long long node_l, long long r, int c) {
    float out[VL];
    const bool ok = tap2_message<DOM, VL, LP, R, O>(a, red, x0, row, out);
    if (!active) return;
    const long long W = a.W;
    const long long step = DIR == 0 ? 1 : DIR == 1 ? -1 : DIR == 2 ? W : -W;
    const long long dir_off = dir_wslot(DIR) * a.slot_stride + step * a.Ms;
    float *dst = it.msgs_out + (node_l * a.Ms + x0) + dir_off;
    if (a.delta)
        *it.dmax = fmaxf(*it.dmax, message_delta<DOM, VL>(out, it.msgs_in + (node_l * a.Ms + x0) + dir_off,
                                                         it.first, x0, a.M));
    Vec8Loader<VL>::store(dst, out);
    if (!ok && j == 0) report_failure(a.err, it.iteration, directed_edge_id(a.H, W, r, c, DIR));
}

// Rows of a node: rows[dir] holds h_{i \ dir's target}; red[dir] its S / H.
template <int DOM, int VL, int LP, bool RX>
__device__ __forceinline__ void tap2_form_h(const float (&g)[VL], const float (&m0)[VL],
                                            const float (&m1)[VL], const float (&m2)[VL],
                                            const float (&m3)[VL], int x0, float *rows,
                                            float (&red)[4]) {
    constexpr int ROWF = TapRow<VL * LP, VL>::PHYS;
    float h[VL];
    if (DOM == SBP_SUM) {
        // reference order: unary, slots 0..3 ascending skipping the excluded
        // one; the same association as band_group_body (bitwise equal)
        vmul(h, g, m1);
        vmul(h, h, m2);
        vmul(h, h, m3);                               // excl 0 -> dir 3
        put_row<DOM, VL, LP>(rows + 3 * ROWF, x0, h);
        red[3] = node_reduce<DOM, VL, LP, RX>(h);
        float ab[VL];
        vmul(ab, g, m0);
        vmul(h, ab, m2);
        vmul(h, h, m3);                               // excl 1 -> dir 1
        put_row<DOM, VL, LP>(rows + 1 * ROWF, x0, h);
        red[1] = node_reduce<DOM, VL, LP, RX>(h);
        vmul(ab, ab, m1);
        vmul(h, ab, m3);                              // excl 2 -> dir 0
        put_row<DOM, VL, LP>(rows + 0 * ROWF, x0, h);
        red[0] = node_reduce<DOM, VL, LP, RX>(h);
        vmul(h, ab, m2);                              // excl 3 -> dir 2
        put_row<DOM, VL, LP>(rows + 2 * ROWF, x0, h);
        red[2] = node_reduce<DOM, VL, LP, RX>(h);
    } else {
        float s2[VL], e2[VL];
        vtwo_sum(g, m1, s2, e2);
        vtwo_sum_acc(s2, m2, e2, e2);
        vtwo_sum_acc(s2, m3, e2, e2);
        shift_compensated<VL, LP, RX>(s2, e2, h);        // excl 0 -> dir 3
        put_row<DOM, VL, LP>(rows + 3 * ROWF, x0, h);
        red[3] = node_reduce<DOM, VL, LP, RX>(h);
        float sa[VL], ea[VL];
        vtwo_sum(g, m0, sa, ea);
        vtwo_sum_from(sa, ea, m2, s2, e2);
        vtwo_sum_acc(s2, m3, e2, e2);
        shift_compensated<VL, LP, RX>(s2, e2, h);        // excl 1 -> dir 1
        put_row<DOM, VL, LP>(rows + 1 * ROWF, x0, h);
        red[1] = node_reduce<DOM, VL, LP, RX>(h);
        vtwo_sum_acc(sa, m1, ea, ea);
        vtwo_sum_from(sa, ea, m3, s2, e2);
        shift_compensated<VL, LP, RX>(s2, e2, h);        // excl 2 -> dir 0
        put_row<DOM, VL, LP>(rows + 0 * ROWF, x0, h);
        red[0] = node_reduce<DOM, VL, LP, RX>(h);
        vtwo_sum_from(sa, ea, m2, s2, e2);
        shift_compensated<VL, LP, RX>(s2, e2, h);        // excl 3 -> dir 2
        put_row<DOM, VL, LP>(rows + 2 * ROWF, x0, h);
        red[2] = node_reduce<DOM, VL, LP, RX>(h);
    }
}

template <int VL, int LP, int STG>
struct Tap2Smem {
    static constexpr int PPW = 32 / LP;
    static constexpr int ROWF = TapRow<VL * LP, VL>::PHYS;
    static constexpr int ROWS_F = (PPW * 4 * ROWF + 31) / 32 * 32;
    static constexpr int STAGE_F = STG == 1 ? 5 * 32 * VL : 0;   // next group's 5 input vectors
    static constexpr int WARP_F = ROWS_F + STAGE_F;
    static constexpr size_t bytes() { return (size_t)TAP_WARPS * WARP_F * sizeof(float); }
};

template <int DOM, int VL, int LP>
__device__ __forceinline__ void tap2_rows_init(float *wbase) {
    using Row = TapRow<VL * LP, VL>;
    constexpr int NROWS = 4 * (32 / LP);
    constexpr float PAD = DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    const int lane = threadIdx.x & 31;
    constexpr int PER = 2 * Row::PADL / 4;   // 4-float pad chunks per row
    for (int k = lane; k < NROWS * PER; k += 32) {
        const int rw = k / PER, q = k % PER;
        const int y = q < Row::PADL / 4 ? 4 * q : Row::PADL + VL * LP + 4 * (q - Row::PADL / 4);
        sts128(wbase + rw * Row::PHYS + Row::phys(y), PAD, PAD, PAD, PAD);
    }
    __syncwarp();
}

#ifndef SBP_TAP2_BLOCKS
#define SBP_TAP2_BLOCKS 8
#endif
// STG = 1: the next pixel group's five input vectors are fetched into shared
// memory by the tensor-memory accelerator (1-D bulk copies on an mbarrier)
// while the current group computes, instead of register loads whose latency
// the first products of the group wait on (ncu: 10-20 % of the samples of the
// register-loaded kernel stall on the first FMUL2 of a group).  STG = 2: the
// register loads stay, and the next group's vectors are prefetched into L2
// (cp.async.bulk.prefetch) one group ahead -- no shared memory, no occupancy
// cost.  STG = 3: register double buffering -- the next group's loads are
// issued right after this group's exclusion vectors are formed and land
// while its four messages are computed (+40 registers: 5 / 4 blocks per SM).
template <int DOM, int VL, int LP, int R, int ROLLED, int STG>
__global__ void __launch_bounds__(32 * TAP_WARPS, (STG == 1 ? 5 : STG == 3 ? (DOM == SBP_SUM ? 5 : 4)
                                                   : (DOM == SBP_SUM ? SBP_TAP2_BLOCKS : 6)))
band_iter_tap2_kernel(const __grid_constant__ BandArgs a) {
    using SM = Tap2Smem<VL, LP, STG>;
    constexpr int PPW = 32 / LP;
    constexpr int ROWF = SM::ROWF;
    constexpr int VEC = 32 * VL;
    float dmax = 0.0f;
    const IterCtx it = iter_of(a, &dmax);
    extern __shared__ __align__(128) float tap_smem[];
    __shared__ __align__(8) unsigned long long bars[TAP_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = lane % LP, q = lane / LP;
    const int x0 = j * VL;
    float *wbase = tap_smem + warp * SM::WARP_F;
    float *rows = wbase + q * 4 * ROWF;
    float *stage = wbase + SM::ROWS_F;
    tap2_rows_init<DOM, VL, LP>(wbase);
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long ngroups = (npix + PPW - 1) / PPW;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    long long grp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nvec = it.first ? 1 : 5;
    auto issue = [&](long long gg) {
        if (lane == 0) {
            const long long p0 = gg * PPW;
            const long long n = npix - p0 < PPW ? npix - p0 : PPW;
            const unsigned bytes = (unsigned)(n * a.Ms * 4);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bars[warp], bytes * nvec);
            bulk_g2s(stage, a.values + ((long long)(a.lr_begin - 1) * a.W + p0) * a.Ms, bytes,
                     &bars[warp]);
            if (!it.first)
                for (int k = 0; k < 4; ++k)
                    bulk_g2s(stage + (1 + k) * VEC,
                             it.msgs_in + k * a.slot_stride + ((long long)a.lr_begin * a.W + p0) * a.Ms,
                             bytes, &bars[warp]);
        }
    };
    auto prefetch_l2 = [&](long long gg) {
        if (lane == 0) {
            const long long p0 = gg * PPW;
            const long long n = npix - p0 < PPW ? npix - p0 : PPW;
            const unsigned bytes = (unsigned)(n * a.Ms * 4);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                             a.values + ((long long)(a.lr_begin - 1) * a.W + p0) * a.Ms),
                         "r"(bytes) : "memory");
            if (!it.first)
                for (int k = 0; k < 4; ++k)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     it.msgs_in + k * a.slot_stride +
                                     ((long long)a.lr_begin * a.W + p0) * a.Ms),
                                 "r"(bytes) : "memory");
        }
    };
    float ng[VL], nm[4][VL];   // STG == 3: the next group's inputs, in flight
    auto load_regs = [&](long long gg) {
        long long pp = gg * PPW + q;
        if (pp >= npix) pp = npix - 1;
        const int lr2 = it.lr_begin + (int)(pp / a.W);
        const int c2 = (int)(pp % a.W);
        Vec8Loader<VL>::load(ng, a.values + ((long long)(lr2 - 1) * a.W + c2) * a.Ms + x0);
        if (!it.first) {
            const float *mi = it.msgs_in + ((long long)lr2 * a.W + c2) * a.Ms + x0;
#pragma unroll
            for (int k = 0; k < 4; ++k) Vec8Loader<VL>::load(nm[k], mi + k * a.slot_stride);
        }
    };
    if constexpr (STG == 3) {
        if (grp < ngroups) load_regs(grp);
    }
    unsigned phase = 0;
    if constexpr (STG == 1) {
        if (lane == 0) {
            mbar_init(&bars[warp], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        if (grp < ngroups) issue(grp);
    }
    for (; grp < ngroups; grp += nwarps) {
        long long p = grp * PPW + q;
        const bool valid = p < npix;
        if (!valid) p = npix - 1;
        const int lr = it.lr_begin + (int)(p / a.W);
        const int c = (int)(p % a.W);
        const long long r = (long long)a.r0 + lr - 1;
        const long long node_l = (long long)lr * a.W + c;
        float red[4];
        {
            float g[VL], m0[VL], m1[VL], m2[VL], m3[VL];
            if constexpr (STG == 2) {
                if (grp + nwarps < ngroups) prefetch_l2(grp + nwarps);
            }
            if constexpr (STG == 3) {
#pragma unroll
                for (int i = 0; i < VL; ++i) {
                    g[i] = ng[i];
                    m0[i] = nm[0][i]; m1[i] = nm[1][i]; m2[i] = nm[2][i]; m3[i] = nm[3][i];
                }
            } else if constexpr (STG == 1) {
                mbar_wait(&bars[warp], phase);
                phase ^= 1u;
                const float *src = stage + q * a.Ms + x0;
                float *mm[5] = {g, m0, m1, m2, m3};
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    if (k > 0 && it.first) break;
#pragma unroll
                    for (int i = 0; i < VL; i += 4) {
                        const float4 v = *reinterpret_cast<const float4 *>(src + k * VEC + i);
                        mm[k][i] = v.x; mm[k][i + 1] = v.y; mm[k][i + 2] = v.z; mm[k][i + 3] = v.w;
                    }
                }
                __syncwarp();   // every lane has its inputs: refill the stage
                if (grp + nwarps < ngroups) issue(grp + nwarps);
            } else {
                Vec8Loader<VL>::load(g, a.values + ((long long)(lr - 1) * a.W + c) * a.Ms + x0);
                if (!it.first) {
                    const float *mi = it.msgs_in + node_l * a.Ms + x0;
                    Vec8Loader<VL>::load(m0, mi);
                    Vec8Loader<VL>::load(m1, mi + a.slot_stride);
                    Vec8Loader<VL>::load(m2, mi + 2 * a.slot_stride);
                    Vec8Loader<VL>::load(m3, mi + 3 * a.slot_stride);
                }
            }
            if (it.first) {
                const bool ghost[4] = {r == 0, c == 0, c == a.W - 1, r == a.H - 1};
                float *mm[4] = {m0, m1, m2, m3};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float real = DOM == SBP_SUM ? (ghost[k] ? 1.0f : 1.0f / (float)a.M) : 0.0f;
#pragma unroll
                    for (int i = 0; i < VL; ++i)
                        mm[k][i] = x0 + i < a.M ? real : (DOM == SBP_SUM ? 0.0f : -__builtin_huge_valf());
                }
            }
            __syncwarp();   // the previous group's messages are done reading the rows
            tap2_form_h<DOM, VL, LP, tap2_redux<DOM, LP, R>()>(g, m0, m1, m2, m3, x0, rows, red);
            if constexpr (STG == 3) {
                if (grp + nwarps < ngroups) load_regs(grp + nwarps);
            }
        }
        __syncwarp();
        const unsigned has = (c + 1 < a.W ? 1u : 0u) | (c > 0 ? 2u : 0u) |
                             (r + 1 < a.H ? 4u : 0u) | (r > 0 ? 8u : 0u);
        auto one = [&](int dir, float rd) {
            const bool hd = (has >> dir) & 1u;
            if (!__any_sync(SBP_FULL_MASK, valid && hd)) return;
            if (ROLLED != 0 || dir == 0 || dir == 2)
                tap2_emit<DOM, VL, LP, R, 0>(a, it, rd, rows + dir * ROWF, dir, j, x0, valid && hd,
                                             node_l, r, c);
            else
                tap2_emit<DOM, VL, LP, R, 1>(a, it, rd, rows + dir * ROWF, dir, j, x0, valid && hd,
                                             node_l, r, c);
        };
        if constexpr (ROLLED == 1) {
#pragma unroll 1
            for (int k = 0; k < 4; ++k) {
                const int dir = (0x2013 >> (4 * k)) & 0xF;   // order 3, 1, 0, 2
                const float rd = dir == 0 ? red[0] : dir == 1 ? red[1] : dir == 2 ? red[2] : red[3];
                one(dir, rd);
            }
        } else if constexpr (ROLLED == 2) {
            // two band copies, a loop of two: half the instruction footprint
            // of the unrolled body (which misses in the instruction cache for
            // wide max-sum bands), half the loop overhead of the rolled one
#pragma unroll 1
            for (int k = 0; k < 2; ++k) {
                one(k ? 0 : 3, k ? red[0] : red[3]);
                one(k ? 2 : 1, k ? red[2] : red[1]);
            }
        } else {
            one(3, red[3]);
            one(1, red[1]);
            one(0, red[0]);
            one(2, red[2]);
        }
    }
    if (a.delta) flush_delta(a.delta, dmax);
}

template <int DOM, int VL, int LP, int R, int ROLLED, int STG>
cudaError_t launch_band_tap2(const BandArgs &a, cudaStream_t s) {
    constexpr int PPW = 32 / LP;
    const size_t smem = Tap2Smem<VL, LP, STG>::bytes();
    static int resident = 0, sms = 0;
    if (!resident) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(band_iter_tap2_kernel<DOM, VL, LP, R, ROLLED, STG>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &resident, band_iter_tap2_kernel<DOM, VL, LP, R, ROLLED, STG>, 32 * TAP_WARPS, smem);
        if (resident < 1) resident = 1;
    }
    const long long npix = (long long)(a.lr_end - a.lr_begin) * a.W;
    const long long warps = (npix + PPW - 1) / PPW;
    long long blocks = (warps + TAP_WARPS - 1) / TAP_WARPS;
    if (blocks <= 0) return cudaSuccess;
    const long long cap = (long long)sms * resident;
    if (blocks > cap) blocks = cap;
    if (launch_block_cap() > 0 && blocks > launch_block_cap()) blocks = launch_block_cap();
    band_iter_tap2_kernel<DOM, VL, LP, R, ROLLED, STG><<<(unsigned)blocks, 32 * TAP_WARPS, smem, s>>>(a);
    return cudaGetLastError();
}

// Radii with a shared-memory-tap kernel (multiples of 4: 4-tap chunks).
// variant: 0 register-loaded, 1 TMA-staged (2 stages), rolled or unrolled.
template <int MS, int DOM>
BandLaunchFn pick_band_tap(int vl, int R, int rolled, int staged) {
    if constexpr (MS < 64) {
        return nullptr;
    } else {
#define SBP_TAP(RR)                                                                          \
    if (R == RR) {                                                                           \
        if (vl == 8 && staged >= 2 && staged <= 5) {                                       \
            const int stg = staged == 2 ? 0 : staged == 3 ? 1 : staged == 4 ? 2 : 3;         \
            const int rl = rolled == 1 ? 1 : rolled == 2 ? 2 : 0;                              \
            if (stg == 0) return rl == 1 ? &launch_band_tap2<DOM, 8, MS / 8, RR, 1, 0>         \
                               : rl == 2 ? &launch_band_tap2<DOM, 8, MS / 8, RR, 2, 0>         \
                                         : &launch_band_tap2<DOM, 8, MS / 8, RR, 0, 0>;        \
            if (stg == 1) return rl == 1 ? &launch_band_tap2<DOM, 8, MS / 8, RR, 1, 1>         \
                                         : &launch_band_tap2<DOM, 8, MS / 8, RR, 0, 1>;        \
            if (stg == 2) return rl == 1 ? &launch_band_tap2<DOM, 8, MS / 8, RR, 1, 2>         \
                               : rl == 2 ? &launch_band_tap2<DOM, 8, MS / 8, RR, 2, 2>         \
                                         : &launch_band_tap2<DOM, 8, MS / 8, RR, 0, 2>;        \
            return rl == 1 ? &launch_band_tap2<DOM, 8, MS / 8, RR, 1, 3>                       \
                 : rl == 2 ? &launch_band_tap2<DOM, 8, MS / 8, RR, 2, 3>                       \
                           : &launch_band_tap2<DOM, 8, MS / 8, RR, 0, 3>;                      \
        }                                                                                    \
        if (vl == 8) {                                                                       \
            if (rolled) return staged ? &launch_band_tap<DOM, 8, MS / 8, RR, true, 2>        \
                                      : &launch_band_tap<DOM, 8, MS / 8, RR, true, 0>;       \
            return staged ? &launch_band_tap<DOM, 8, MS / 8, RR, false, 2>                   \
                          : &launch_band_tap<DOM, 8, MS / 8, RR, false, 0>;                  \
        }                                                                                    \
        if constexpr (MS >= 128 && DOM == SBP_SUM) {                                         \
            if (vl == 16 && !staged)                                                         \
                return rolled ? &launch_band_tap<DOM, 16, MS / 16, RR, true, 0>              \
                              : &launch_band_tap<DOM, 16, MS / 16, RR, false, 0>;            \
        }                                                                                    \
        return nullptr;                                                                      \
    }
        SBP_TAP(8)
        SBP_TAP(16)
        SBP_TAP(32)
#undef SBP_TAP
        return nullptr;
    }
}

}  // namespace sbp
