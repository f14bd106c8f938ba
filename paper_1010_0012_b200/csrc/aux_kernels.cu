// Bookkeeping kernels around the message kernel: message init, value upload,
// beliefs / MAP labels, directed-edge store gather, convergence delta.
#include "aux_kernels.cuh"

namespace sbp {

// bp.py:587-601: sum -> 1/M on real slots and 1 on ghost slots (no
// neighbour: the product identity, so border nodes need no branches);
// max -> 0.  Labels >= M are padding: 0 (sum) / -inf (max).
__global__ void init_msgs_kernel(float *msgs, int H, int W, int M, int Ms, int r0, int rows,
                                 int domain) {
    const long long per_slot = (long long)(rows + 2) * W * Ms;
    const long long total = 4 * per_slot;
    const float uni = 1.0f / (float)M;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % Ms);
        const long long node = (i / Ms) % ((long long)(rows + 2) * W);
        const int k = (int)(i / per_slot);
        const int c = (int)(node % W);
        const long long r = (long long)r0 + node / W - 1;
        float v;
        if (x >= M) {
            v = domain == SBP_SUM ? 0.0f : -__builtin_huge_valf();
        } else if (domain == SBP_MAX) {
            v = 0.0f;
        } else {
            const bool ghost = (k == 0 && r <= 0) || (k == 1 && c == 0) ||
                               (k == 2 && c == W - 1) || (k == 3 && r >= H - 1);
            v = ghost ? 1.0f : uni;
        }
        msgs[i] = v;
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

// One warp per node, lanes stride the labels.  Sum: b = g * m0 * m1 * m2 * m3
// in the order np.multiply.at applies them (bp.py:715-720; ghost slots are
// exactly 1), rescaled by the running max after every factor so fp32 does
// not underflow on peaked messages, Z = sum * prod(scales) in
// f64, beliefs = b / sum.  Max: s = ln g + m0 + m1 + m2 + m3 - max
// (bp.py:728-738).  Labels: argmax, lowest index on ties (bp.py:741-744).
template <int DOM>
__global__ void beliefs_kernel(const float *values, const float *msgs, int W, int M, int Ms,
                               int rows, float *beliefs, double *normalizers, int *labels,
                               unsigned long long *bad_node) {
    const long long slot = (long long)(rows + 2) * W * Ms;
    const int lane = threadIdx.x & 31;
    const long long nodes = (long long)rows * W;
    const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long n = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; n < nodes;
         n += warps) {
        const float *g = values + n * Ms;
        const float *m = msgs + (n + W) * Ms;   // local row = global row + 1
        double scale = 1.0;
        float z = 0.0f, best = -__builtin_huge_valf();
        int best_x = 0x7fffffff;
        if (DOM == SBP_SUM) {
            // pass 1: per-label product with rescaling; each lane keeps its labels
            // in registers only for Ms <= 256 (8 per lane)
            float b[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int x = lane + 32 * q;
                b[q] = (x < M) ? g[x] : 0.0f;
            }
            for (int k = 0; k < 4; ++k) {
                float mx = 0.0f;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int x = lane + 32 * q;
                    if (x < M) b[q] *= m[k * slot + x];
                    mx = fmaxf(mx, b[q]);
                }
                for (int off = 16; off; off >>= 1)
                    mx = fmaxf(mx, __shfl_xor_sync(SBP_FULL_MASK, mx, off));
                // rescale by an exact power of two so the running max stays
                // in [1, 2): no rounding, no drift towards the denormals
                if (mx > 0.0f) {
                    int e;
                    frexpf(mx, &e);
                    e -= 1;
                    if (e != 0) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) b[q] = ldexpf(b[q], -e);
                        scale = ldexp(scale, e);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) z += b[q];
            for (int off = 16; off; off >>= 1) z += __shfl_xor_sync(SBP_FULL_MASK, z, off);
            if (!(z > 0.0f)) {
                if (lane == 0 && bad_node) atomicMin(bad_node, (unsigned long long)n);
                continue;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int x = lane + 32 * q;
                if (x < M) {
                    const float v = b[q] / z;
                    if (beliefs) beliefs[n * M + x] = v;
                    if (v > best) { best = v; best_x = x; }
                }
            }
            if (lane == 0 && normalizers) normalizers[n] = (double)z * scale;
        } else {
            // scores in f64: ln g + m0 + m1 + m2 + m3 - max, rounded once
            double s[8];
            double mx = -__builtin_huge_val();
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int x = lane + 32 * q;
                if (x < M) {
                    double v = (double)g[x];
                    for (int k = 0; k < 4; ++k) v += (double)m[k * slot + x];
                    s[q] = v;
                    mx = fmax(mx, v);
                } else {
                    s[q] = -__builtin_huge_val();
                }
            }
            for (int off = 16; off; off >>= 1)
                mx = fmax(mx, __shfl_xor_sync(SBP_FULL_MASK, mx, off));
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int x = lane + 32 * q;
                if (x < M) {
                    const float v = (float)(s[q] - mx);
                    if (beliefs) beliefs[n * M + x] = v;
                    if (v > best) { best = v; best_x = x; }
                }
            }
        }
        // argmax across lanes: larger value wins, lower label on ties
        for (int off = 16; off; off >>= 1) {
            const float ov = __shfl_xor_sync(SBP_FULL_MASK, best, off);
            const int ox = __shfl_xor_sync(SBP_FULL_MASK, best_x, off);
            if (ov > best || (ov == best && ox < best_x)) { best = ov; best_x = ox; }
        }
        if (lane == 0 && labels) labels[n] = best_x == 0x7fffffff ? 0 : best_x;
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
                             int domain, cudaStream_t s) {
    init_msgs_kernel<<<grid_for(4LL * (rows + 2) * W * Ms, 256), 256, 0, s>>>(
        msgs, H, W, M, Ms, r0, rows, domain);
    return cudaGetLastError();
}

cudaError_t launch_load_values(const double *src, float *dst, long long nodes, int M, int Ms,
                               int domain, cudaStream_t s) {
    load_values_kernel<<<grid_for(nodes * 32, 256), 256, 0, s>>>(src, dst, nodes, M, Ms, domain);
    return cudaGetLastError();
}

cudaError_t launch_beliefs(int domain, const float *values, const float *msgs, int W, int M,
                           int Ms, int rows, float *beliefs, double *normalizers, int *labels,
                           unsigned long long *bad_node, cudaStream_t s) {
    const unsigned blocks = grid_for((long long)rows * W * 32, 256);
    if (domain == SBP_SUM)
        beliefs_kernel<SBP_SUM><<<blocks, 256, 0, s>>>(values, msgs, W, M, Ms, rows, beliefs,
                                                       normalizers, labels, bad_node);
    else
        beliefs_kernel<SBP_MAX><<<blocks, 256, 0, s>>>(values, msgs, W, M, Ms, rows, beliefs,
                                                       normalizers, labels, bad_node);
    return cudaGetLastError();
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
