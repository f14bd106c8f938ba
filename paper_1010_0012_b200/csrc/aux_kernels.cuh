#pragma once
#include "sbp_common.cuh"

namespace sbp {

cudaError_t launch_init_msgs(float *msgs, int H, int W, int M, int Ms, int r0, int rows,
                             int domain, int ghosts_only, cudaStream_t s);
cudaError_t launch_load_values(const double *src, float *dst, long long nodes, int M, int Ms,
                               int domain, cudaStream_t s);
cudaError_t launch_beliefs(int domain, const float *values, const float *msgs, int W, int M,
                           int Ms, int rows, float *beliefs, double *normalizers, int *labels,
                           unsigned long long *bad_node, cudaStream_t s);
cudaError_t launch_gather_store(const float *msgs, int H, int W, int M, int Ms, float *out,
                                cudaStream_t s);
cudaError_t launch_stereo_values(const unsigned char *left, const unsigned char *right,
                                 long long rows, int W, int M, int Ms, double beta, double T_u,
                                 int domain, float *dst, cudaStream_t s);
cudaError_t launch_max_abs_diff(const float *a, const float *b, int W, int M, int Ms, int rows,
                                float *out, cudaStream_t s);

struct EllArgs {
    const float *values;
    const float *msgs_in;
    float *msgs_out;
    unsigned long long *err;
    long long slot_stride;
    int H, W, M, Ms, r0, lr_begin, lr_end, iteration, floor_term, m_max;
    int first, pass;
    float fbar[2];              // shared potential: per orientation
    const int *idx;             // [n_pot][2][m_max][Ms]
    const float *w;             // [n_pot][2][m_max][Ms]
    long long pot_stride;       // m_max * Ms
    const float *fbar_all;      // per-edge: [n_pot][2], else NULL
    const int *pid_h, *pid_v;   // per-edge potential ids (global nodes), else NULL
    int acc64;                  // sum-product in f64 (sbp_potential::accumulate)
    double fbar64[2];
    const float *w_lo;          // acc64: low f32 plane of the weights (w = w + w_lo)
    float *delta;               // fused convergence test (BandArgs::delta), NULL: off
};
cudaError_t launch_ell(int domain, const EllArgs &a, cudaStream_t s);
cudaError_t launch_ell_sweep(int domain, const EllArgs &a, cudaStream_t s);

struct DenseArgs {
    const float *values;
    const float *msgs_in;
    float *msgs_out;
    unsigned long long *err;
    long long slot_stride;
    int H, W, M, Ms, r0, lr_begin, lr_end, iteration, first;
    const float *t[2];   // [Ms][Ms] per orientation: f(x_i = k, x_j = x) at [k][x]
};
cudaError_t launch_dense(int domain, const DenseArgs &a, cudaStream_t s);
// Sum-product, symmetric table (t[0] serves both orientations), Ms = 128 or
// 256: the same update as a 3xTF32 GEMM on the tensor cores (dense_tc_kernel.cu).
bool dense_tc_supported(int Ms);
cudaError_t launch_dense_tc(const DenseArgs &a, bool bf16_corrections, cudaStream_t s);



}  // namespace sbp
