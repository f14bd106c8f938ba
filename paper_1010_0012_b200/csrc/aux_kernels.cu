// Bookkeeping kernels around the message kernel: message init, value upload,
// beliefs / MAP labels, directed-edge store gather, convergence delta.
#include "aux_kernels.cuh"
#include "band_kernel.cuh"   // Vec8Loader, lanes_sum / lanes_max

namespace sbp {

// bp.py:587-601: sum -> 1/M on real slots and 1 on ghost slots (no
// neighbour: the product identity, so border nodes need no branches);
// max -> 0.  Labels >= M are padding: 0 (sum) / -inf (max).  One warp per
// node vector, 16-byte stores.  With ghosts_only the warp list is just the
// border slots (2W + 2 rows vectors): the message kernels never write them
// and overwrite every real slot, so this is all a buffer needs once.
__global__ void init_msgs_kernel(float *msgs, int H, int W, int M, int Ms, int r0, int rows,
                                 int domain, int ghosts_only) {
    const long long per_slot = (long long)(rows + 2) * W;   // node vectors per slot
    const long long count = ghosts_only ? 2LL * W + 2LL * rows : 4 * per_slot;
    const int lane = threadIdx.x & 31;
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    const float pad = domain == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    const bool top = r0 == 0, bottom = r0 + rows == H;
    for (long long v = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < count;
         v += warps) {
        int k;
        long long lr, c;
        if (!ghosts_only) {
            k = (int)(v / per_slot);
            lr = (v % per_slot) / W;
            c = v % W;
        } else if (v < W) {                       // slot 0, global row 0
            if (!top) continue;
            k = 0; lr = 1; c = v;
        } else if (v < 2LL * W) {                 // slot 3, global row H-1
            if (!bottom) continue;
            k = 3; lr = rows; c = v - W;
        } else if (v < 2LL * W + rows) {          // slot 1, column 0
            k = 1; lr = 1 + (v - 2LL * W); c = 0;
        } else {                                  // slot 2, column W-1
            k = 2; lr = 1 + (v - 2LL * W - rows); c = W - 1;
        }
        const long long r = (long long)r0 + lr - 1;
        const bool ghost = (k == 0 && r <= 0) || (k == 1 && c == 0) ||
                           (k == 2 && c == W - 1) || (k == 3 && r >= H - 1);
        const float real = domain == SBP_MAX ? 0.0f : (ghost ? 1.0f : 1.0f / (float)M);
        float4 *dst = reinterpret_cast<float4 *>(msgs + (k * per_slot + lr * W + c) * Ms);
        for (int q = lane; q < Ms / 4; q += 32) {
            const int x = 4 * q;
            float4 val;
            val.x = x + 0 < M ? real : pad;
            val.y = x + 1 < M ? real : pad;
            val.z = x + 2 < M ? real : pad;
            val.w = x + 3 < M ? real : pad;
            dst[q] = val;
        }
    }
}

// f64 model values -> padded f32 device table, one warp per node.  In the
// max domain each node's log unary is shifted by its own maximum (computed
// and subtracted in f64): every message is max-normalised and the
// max-marginals subtract the row max, so a per-node constant changes no
// result, but it keeps the magnitudes entering the fp32 h sums small.
__global__ void load_values_kernel(const double *src, float *dst, long long nodes, int M, int Ms,
                                   int domain) {
    const int lane = threadIdx.x & 31;
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long n = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; n < nodes;
         n += warps) {
        const double *s = src + n * M;
        double shift = 0.0;
        if (domain == SBP_MAX) {
            double mx = -__builtin_huge_val();
            for (int x = lane; x < M; x += 32) mx = fmax(mx, s[x]);
            for (int off = 16; off; off >>= 1)
                mx = fmax(mx, __shfl_xor_sync(SBP_FULL_MASK, mx, off));
            if (isfinite(mx)) shift = mx;
        }
        float *d = dst + n * Ms;
        for (int x = lane; x < Ms; x += 32)
            d[x] = x < M ? (float)(s[x] - shift)
                         : (domain == SBP_SUM ? 0.0f : -__builtin_huge_valf());
    }
}

// Beliefs / max-marginals / labels.  LP lanes per node, 8 consecutive labels
// per lane (LP * 8 = Ms), all five input vectors loaded up front with 256-bit
// loads.  Sum: b = g * m0 * m1 * m2 * m3 in the order np.multiply.at applies
// them (bp.py:715-720; ghost slots hold exactly 1), after every factor
// rescaled by an exact power of two so the running max stays in [1, 2) (no
// rounding, no underflow on peaked messages); Z = sum * 2^e in
// f64; beliefs = b / sum.  Max: ln g + m0 + m1 + m2 + m3 - max in f64
// (bp.py:728-738), rounded once.  Labels: argmax, lowest index on ties
// (bp.py:741-744), taken on the values that are returned.
template <int DOM, int LP>
__global__ void __launch_bounds__(256) beliefs_kernel(const float *values, const float *msgs,
                                                      int W, int M, int Ms, int rows,
                                                      float *beliefs, double *normalizers,
                                                      int *labels, unsigned long long *bad_node) {
    constexpr int VL = 8;
    const long long slot = (long long)(rows + 2) * W * Ms;
    const int lane = threadIdx.x & 31;
    const int j = lane % LP;
    const int x0 = j * VL;
    const long long nodes = (long long)rows * W;
    const long long groups = (nodes + (32 / LP) - 1) / (32 / LP);
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < groups;
         w += warps) {
        long long n = w * (32 / LP) + lane / LP;
        const bool valid = n < nodes;
        if (!valid) n = nodes - 1;
        float g[VL], m[4][VL];
        Vec8Loader<VL>::load(g, values + n * Ms + x0);
        const float *mp = msgs + (n + W) * Ms + x0;   // local row = global row + 1
#pragma unroll
        for (int k = 0; k < 4; ++k) Vec8Loader<VL>::load(m[k], mp + k * slot);
        float best = -__builtin_huge_valf();
        int best_x = 0x7fffffff;
        float out[VL];
        if (DOM == SBP_SUM) {
            float b[VL];
            int e_tot = 0;
#pragma unroll
            for (int i = 0; i < VL; ++i) b[i] = g[i];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float mx = 0.0f;
#pragma unroll
                for (int i = 0; i < VL; ++i) {
                    b[i] *= m[k][i];
                    mx = fmaxf(mx, b[i]);
                }
                mx = lanes_max<LP>(mx);
                if (mx > 0.0f) {
                    int e;
                    frexpf(mx, &e);
                    e -= 1;
                    if (e != 0) {
#pragma unroll
                        for (int i = 0; i < VL; ++i) b[i] = ldexpf(b[i], -e);
                        e_tot += e;
                    }
                }
            }
            float z = 0.0f;
#pragma unroll
            for (int i = 0; i < VL; ++i) z += b[i];
            z = lanes_sum<LP>(z);
            if (!(z > 0.0f)) {
                if (valid && j == 0 && bad_node) atomicMin(bad_node, (unsigned long long)n);
                continue;
            }
#pragma unroll
            for (int i = 0; i < VL; ++i) out[i] = b[i] / z;
            if (valid && j == 0 && normalizers) normalizers[n] = ldexp((double)z, e_tot);
        } else {
            double sd[VL];
            double mx = -__builtin_huge_val();
#pragma unroll
            for (int i = 0; i < VL; ++i) {
                double v = (double)g[i];
#pragma unroll
                for (int k = 0; k < 4; ++k) v += (double)m[k][i];
                sd[i] = v;
                if (x0 + i < M) mx = fmax(mx, v);
            }
#pragma unroll
            for (int off = 1; off < LP; off <<= 1)
                mx = fmax(mx, __shfl_xor_sync(SBP_FULL_MASK, mx, off));
#pragma unroll
            for (int i = 0; i < VL; ++i) out[i] = (float)(sd[i] - mx);
        }
#pragma unroll
        for (int i = 0; i < VL; ++i) {
            const int x = x0 + i;
            if (x < M) {
                if (valid && beliefs) beliefs[n * M + x] = out[i];
                if (out[i] > best) { best = out[i]; best_x = x; }
            }
        }
#pragma unroll
        for (int off = 1; off < LP; off <<= 1) {
            const float ov = __shfl_xor_sync(SBP_FULL_MASK, best, off);
            const int ox = __shfl_xor_sync(SBP_FULL_MASK, best_x, off);
            if (ov > best || (ov == best && ox < best_x)) { best = ov; best_x = ox; }
        }
        if (valid && j == 0 && labels) labels[n] = best_x == 0x7fffffff ? 0 : best_x;
    }
}

// Directed id d -> (edge e = d/2, orientation d%2) -> source slot (bp.py:604-617).
__global__ void gather_store_kernel(const float *msgs, int H, int W, int M, int Ms,
                                    float *out) {
    const long long slot = (long long)(H + 2) * W * Ms;
    const long long E = (long long)H * (W - 1) + (long long)W * (H - 1);
    const int lane = threadIdx.x & 31;
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long d = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; d < 2 * E;
         d += warps) {
        const long long e = d >> 1;
        long long r = e / (2LL * W - 1);
        if (r > H - 1) r = H - 1;
        const long long o = e - r * (2LL * W - 1);
        long long c;
        bool horiz;
        if (r < H - 1) {
            if (o < 2LL * (W - 1)) { c = o >> 1; horiz = (o & 1) == 0; }
            else { c = W - 1; horiz = false; }
        } else {
            c = o; horiz = true;
        }
        const long long a = r * W + c;
        const long long b = a + (horiz ? 1 : W);
        int k;
        long long node;
        if ((d & 1) == 0) { k = horiz ? 1 : 0; node = b; }   // a -> b, stored at b
        else { k = horiz ? 2 : 3; node = a; }                 // b -> a, stored at a
        const float *src = msgs + k * slot + (node + W) * Ms;
        for (int x = lane; x < M; x += 32) out[d * M + x] = src[x];
    }
}

__global__ void max_abs_diff_kernel(const float *a, const float *b, int W, int M, int Ms,
                                    int rows, float *out) {
    const long long slot = (long long)(rows + 2) * W * Ms;
    const long long per = (long long)rows * W * Ms;
    float d = 0.0f;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < 4 * per;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(i / per);
        const long long off = i % per;
        if ((int)(off % Ms) >= M) continue;
        const long long idx = k * slot + (long long)W * Ms + off;
        const float v = fabsf(a[idx] - b[idx]);
        d = (v > d || v != v) ? v : d;
    }
    for (int o = 16; o; o >>= 1) {
        const float t = __shfl_xor_sync(SBP_FULL_MASK, d, o);
        d = (t > d || t != t) ? t : d;
    }
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned int *)out, __float_as_uint(d));
}

// -------------------------------------------------------------------------

static unsigned grid_for(long long work, int block) {
    long long b = (work + block - 1) / block;
    if (b > 148LL * 32) b = 148LL * 32;
    return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_init_msgs(float *msgs, int H, int W, int M, int Ms, int r0, int rows,
                             int domain, int ghosts_only, cudaStream_t s) {
    const long long vecs = ghosts_only ? 2LL * W + 2LL * rows : 4LL * (rows + 2) * W;
    init_msgs_kernel<<<grid_for(vecs * 32, 256), 256, 0, s>>>(msgs, H, W, M, Ms, r0, rows,
                                                              domain, ghosts_only);
    return cudaGetLastError();
}

cudaError_t launch_load_values(const double *src, float *dst, long long nodes, int M, int Ms,
                               int domain, cudaStream_t s) {
    load_values_kernel<<<grid_for(nodes * 32, 256), 256, 0, s>>>(src, dst, nodes, M, Ms, domain);
    return cudaGetLastError();
}

template <int DOM>
static cudaError_t launch_beliefs_dom(const float *values, const float *msgs, int W, int M,
                                      int Ms, int rows, float *beliefs, double *normalizers,
                                      int *labels, unsigned long long *bad_node, cudaStream_t s) {
    const long long lanes = (long long)rows * W * (Ms / 8);
    const unsigned blocks = grid_for(lanes, 256);
#define SBP_B(LPV)                                                                        \
    case LPV:                                                                             \
        beliefs_kernel<DOM, LPV><<<blocks, 256, 0, s>>>(values, msgs, W, M, Ms, rows,     \
                                                        beliefs, normalizers, labels, bad_node); \
        break;
    switch (Ms / 8) {
        SBP_B(1) SBP_B(2) SBP_B(4) SBP_B(8) SBP_B(16) SBP_B(32)
    default: return cudaErrorInvalidValue;
    }
#undef SBP_B
    return cudaGetLastError();
}

cudaError_t launch_beliefs(int domain, const float *values, const float *msgs, int W, int M,
                           int Ms, int rows, float *beliefs, double *normalizers, int *labels,
                           unsigned long long *bad_node, cudaStream_t s) {
    if (domain == SBP_SUM)
        return launch_beliefs_dom<SBP_SUM>(values, msgs, W, M, Ms, rows, beliefs, normalizers,
                                           labels, bad_node, s);
    return launch_beliefs_dom<SBP_MAX>(values, msgs, W, M, Ms, rows, beliefs, normalizers,
                                       labels, bad_node, s);
}

cudaError_t launch_gather_store(const float *msgs, int H, int W, int M, int Ms, float *out,
                                cudaStream_t s) {
    const long long E = (long long)H * (W - 1) + (long long)W * (H - 1);
    if (E <= 0) return cudaSuccess;
    gather_store_kernel<<<grid_for(2 * E * 32, 256), 256, 0, s>>>(msgs, H, W, M, Ms, out);
    return cudaGetLastError();
}

cudaError_t launch_max_abs_diff(const float *a, const float *b, int W, int M, int Ms, int rows,
                                float *out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float), s);
    if (e != cudaSuccess) return e;
    max_abs_diff_kernel<<<grid_for(4LL * rows * W * Ms, 256), 256, 0, s>>>(a, b, W, M, Ms,
                                                                          rows, out);
    return cudaGetLastError();
}

}  // namespace sbp

namespace sbp {

// Stereo unary field on the device (reference stereo.py:82-99, 120-125; the
// SURVEY 8f #3 "GPU unary builder"): node (r, c) of the right image, label x:
//     energy = beta * min(|R(r, c) - L(r, c + x)|, T_u)   (c + x < W)
//              beta * T_u                                  (out of frame)
// sum: exp(-energy); max: -energy shifted by the node's max -- computed in
// f64 like the reference, rounded once to f32.  One warp per node.
__global__ void stereo_values_kernel(const unsigned char *left, const unsigned char *right,
                                     long long rows, int W, int M, int Ms, double beta,
                                     double T_u, int domain, float *dst) {
    const int lane = threadIdx.x & 31;
    const long long nodes = rows * W;
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long n = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; n < nodes;
         n += warps) {
        const long long r = n / W;
        const int c = (int)(n % W);
        const int rv = right[r * W + c];
        const unsigned char *lrow = left + r * W;
        const double full = beta * T_u;
        double emin = __builtin_huge_val();
        if (domain == SBP_MAX) {
            for (int x = lane; x < M; x += 32) {
                const double e = c + x < W ? beta * fmin((double)abs(rv - (int)lrow[c + x]), T_u)
                                           : full;
                emin = fmin(emin, e);
            }
            for (int off = 16; off; off >>= 1)
                emin = fmin(emin, __shfl_xor_sync(SBP_FULL_MASK, emin, off));
        }
        float *d = dst + n * Ms;
        for (int x = lane; x < Ms; x += 32) {
            float v;
            if (x >= M) {
                v = domain == SBP_SUM ? 0.0f : -__builtin_huge_valf();
            } else {
                const double e = c + x < W ? beta * fmin((double)abs(rv - (int)lrow[c + x]), T_u)
                                           : full;
                v = domain == SBP_SUM ? (float)exp(-e) : (float)(-e - (-emin));
            }
            d[x] = v;
        }
    }
}

cudaError_t launch_stereo_values(const unsigned char *left, const unsigned char *right,
                                 long long rows, int W, int M, int Ms, double beta, double T_u,
                                 int domain, float *dst, cudaStream_t s) {
    long long b = (rows * W * 32 + 255) / 256;
    if (b > 148LL * 32) b = 148LL * 32;
    stereo_values_kernel<<<(unsigned)(b < 1 ? 1 : b), 256, 0, s>>>(left, right, rows, W, M, Ms,
                                                                   beta, T_u, domain, dst);
    return cudaGetLastError();
}

}  // namespace sbp
