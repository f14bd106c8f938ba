/*
 * sbp.h -- C ABI of the B200 grid loopy-BP engine (libsbp.so).
 *
 * Plain pointers and sizes only; every device pointer is caller-owned
 * (the library never allocates or frees caller memory) and every call is
 * stream-ordered on the caller's `cudaStream_t` (passed as void*).
 *
 * Each entry point replaces one piece of the reference `sparsebp` grid
 * engine (/root/reference/pkg/src/sparsebp):
 *
 *   sbp_init_msgs      <- bp.py:587-601      `_grid_store_init`
 *   sbp_load_values    <- bp.py:488          values_in = unaries | log_unaries
 *                                            (f64 host model -> padded f32 device)
 *   sbp_stereo_values  <- stereo.py:82-99,120-125 unary field on the device
 *   sbp_iterate        <- bp.py:492-503 + numba_kernels.py:296-316,364-384
 *                         (`_run_grid` -> `grid_pass_{sum,max}_{fast,standard,pruned}`);
 *                         one SYNCHRONOUS iteration of all directed updates
 *                         of a row range: _grid_h_* (:194-227) -> _fast_* /
 *                         _std_* / _pruned_* (:35-101) -> _norm_*_store (:248-271)
 *   sbp_iterate_fused  <- bp.py:660-676 (the run_sweeps loop): 1..4 consecutive
 *                         synchronous iterations in one launch (sbp_iterate's
 *                         arithmetic, intermediate messages kept in L2)
 *   sbp_sweep          <- bp.py:492-503 + numba_kernels.py:274-407: one canonical
 *                         sequential sweep (the reference default schedule)
 *   sbp_beliefs        <- bp.py:711-744      `compute_beliefs`,
 *                                            `compute_max_marginals`, `map_labels`
 *   sbp_gather_store   <- bp.py:604-617      `_grid_store_to_messages`
 *   sbp_max_abs_diff   <- bp.py:671-676      convergence test of `run_sweeps`
 *                         (sbp_iterate_delta / sbp_sweep_delta fuse it into the
 *                         iteration; this separate pass serves the dense kernel)
 *
 * Device layout:
 *   values  [rows][W][Ms]          f32, labels >= M padded (0 sum / -inf max)
 *   msgs    [4][rows+2][W][Ms]     f32; local row lr <-> global row r0+lr-1,
 *                                  rows 0 and rows+1 are halo rows; slot k holds
 *                                  the message INTO the node from direction k
 *                                  (0 above, 1 left, 2 right, 3 below).
 * Errors: every function returns SBP_OK or a negative code; the text of
 * the last error of the calling thread is available from sbp_last_error().
 * A message that cannot be normalised (reference DegenerateMessageError,
 * bp.py:499-503) is reported through the device word `err`:
 * min over failures of (iteration << 40 | reference directed-edge id).
 */
#ifndef SBP_H
#define SBP_H

#include <stdint.h>

#if defined(__GNUC__)
#define SBP_API __attribute__((visibility("default")))
#else
#define SBP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SBP_OK 0
#define SBP_EINVAL (-1)
#define SBP_ECUDA (-2)
#define SBP_EUNSUPPORTED (-3)

#define SBP_SUM 0
#define SBP_MAX 1

#define SBP_POT_BAND 0   /* Toeplitz band |x_i - x_j| <= R, weights in kernel params */
#define SBP_POT_ELL 1    /* general per-column lists (ELL [m_max][Ms]) */
#define SBP_POT_DENSE 2  /* dense O(M^2) comparison kernel (reference "standard") */

#define SBP_MAX_R 32
#define SBP_ERR_NONE 0xffffffffffffffffull

#define SBP_DEVICE_AUTO (-1)

typedef struct {
    int H, W;      /* global grid */
    int M, Ms;     /* labels and padded per-node stride (multiple of 4) */
    int r0, rows;  /* this strip: global rows r0 .. r0+rows-1 */
    int device;    /* CUDA device owning every buffer passed with this grid; the
                      library (static CUDA runtime) selects it before launching.
                      SBP_DEVICE_AUTO: look it up from the buffer pointers
                      (cudaPointerGetAttributes on every call). */
} sbp_grid;

typedef struct {
    int kind;            /* SBP_POT_* */
    int domain;          /* SBP_SUM | SBP_MAX */
    int floor_term;      /* 1: reference "fast" (fbar branch), 0: "pruned" */
    int R;               /* BAND: radius, weights for d = x_i - x_j in [-R, R] */
    int m_max;           /* ELL: entries per column */
    float fbar[2];       /* per orientation: fbar (sum) or ln fbar (max) */
    float band_w[2][2 * SBP_MAX_R + 1];   /* BAND: w[o][d + R] (residual | log value) */
    const int32_t *ell_idx[2];            /* ELL: device [m_max][Ms] per orientation, x_i per
                                             (k, x_j); ell_idx[1] == ell_idx[0] + m_max*Ms */
    const float *ell_w[2];                /* ELL: device [m_max][Ms], same layout */
    const float *dense_t[2];              /* DENSE: device [Ms][Ms] per orientation,
                                             f(x_i = k, x_j = x) at [k][x] (tiled kernel,
                                             Ms >= 32); smaller Ms runs the ELL arrays with
                                             m_max = M, idx[k][x] = k.  A symmetric table may
                                             pass the SAME pointer twice: sum-product at
                                             Ms = 128 / 256 then runs as a 3xTF32 GEMM on the
                                             tensor cores (tcgen05; SBP_DENSE_TC=0: SIMT,
                                             2: bf16 correction products, faster, 5.7e-6) */
    /* ELL per-edge (inhomogeneous) potentials, n_pot > 0: ell_idx[0] / ell_w[0]
     * point at [n_pot][2][m_max][Ms], fbar_all at [n_pot][2]; pid_h[r*W + c]
     * is the potential of edge (n, n+1), pid_v[r*W + c] of edge (n, n+W)
     * (global node n = r*W + c).  n_pot = 0: one shared potential. */
    int n_pot;
    const float *fbar_all;
    const int32_t *pid_h;
    const int32_t *pid_v;
    /* Accumulation precision of sum-product (SBP_ACC_*): SBP_ACC_F64 computes
     * products, sums and the normaliser in f64 from the f32-stored messages
     * (reference precision, numba_kernels.py:44-54); ELL kind, shared potential
     * only; the weights then carry f64 precision as ell_w (high f32 plane) +
     * ell_w_lo (low plane) and fbar as fbar64. */
    int accumulate;
    double fbar64[2];
    const float *ell_w_lo[2];
} sbp_potential;

#define SBP_ACC_F32 0
#define SBP_ACC_F64 1

SBP_API int sbp_version(void);
SBP_API const char *sbp_last_error(void);

/* The SBP_* environment knobs (kernel-variant overrides for A/B runs) are read
 * once per process; this re-reads them. */
SBP_API int sbp_reload_config(void);

/* Padded label stride the band kernels use for M labels (>= M, multiple of 4). */
SBP_API int sbp_padded_labels(int M);

/* Compiled band radius a Toeplitz band of radius R runs on at padded stride
 * Ms (the smallest compiled radius >= R that is < Ms), or 0 when no band
 * kernel exists -- the host then plans the general ELL kernel instead
 * (reference numba_kernels.py:44-54 runs any CSC; bp.py:466-489). */
SBP_API int sbp_band_radius(int Ms, int R);

/* Initial messages (bp.py:587-601).  ghosts_only = 1 writes only the border
 * (ghost) slots, which the iteration kernels never write: enough for a fresh
 * buffer when the first iteration runs with SBP_ITER_FIRST. */
SBP_API int sbp_init_msgs(const sbp_grid *g, int domain, int ghosts_only, float *msgs,
                          void *stream);

/* f64 [rows][W][M] (device) -> padded f32 values [rows][W][Ms]. */
SBP_API int sbp_load_values(const sbp_grid *g, int domain, const double *src, float *dst, void *stream);

/* Stereo unaries straight from the image pair (stereo.py:82-99,120-125):
 * left/right are device [rows][W] uint8 of this strip's rows; dst as in
 * sbp_load_values (sum: exp(-energy); max: -energy shifted by the node max). */
SBP_API int sbp_stereo_values(const sbp_grid *g, int domain, const uint8_t *left,
                              const uint8_t *right, double beta, double T_u, float *dst,
                              void *stream);

/* One synchronous iteration over local rows [lr_begin, lr_end) (1-based
 * strip rows; a full grid is r0 = 0, rows = H, lr in [1, H+1)).  With
 * SBP_ITER_FIRST in flags the incoming messages are taken to be the
 * reference initial messages and msgs_in is not read. */
#define SBP_ITER_FIRST 1
SBP_API int sbp_iterate(const sbp_grid *g, const sbp_potential *pot, const float *values,
                        const float *msgs_in, float *msgs_out, int lr_begin, int lr_end,
                        int iteration, int flags, unsigned long long *err, void *stream);

/* sbp_iterate with the convergence test of run_sweeps fused in (bp.py:671-676,
 * `delta = |msgs4 - prev|.max()`): every written message is compared with
 * the value it replaces (msgs_in at the same slot; the reference initial
 * message at iteration 0) and *delta (device float, zeroed by the caller)
 * is max-updated.  The old values are the ones the neighbouring nodes read
 * in the same pass, so they come from L2, not a second HBM pass.  Band and
 * ELL potentials; the dense comparison kernel returns SBP_EUNSUPPORTED. */
SBP_API int sbp_iterate_delta(const sbp_grid *g, const sbp_potential *pot, const float *values,
                              const float *msgs_in, float *msgs_out, int lr_begin, int lr_end,
                              int iteration, int flags, unsigned long long *err, float *delta,
                              void *stream);

/* `levels` (1..4) consecutive synchronous iterations over the whole strip in
 * ONE persistent cooperative launch (temporal blocking: a row wavefront with
 * `lag` rows between levels; the intermediate messages stay in L2 and are
 * discarded there once read).  Level l reads buffer l % 2 of (msgs_a, msgs_b)
 * and writes the other: the result is in msgs_a for even `levels`, msgs_b
 * for odd; the intermediate buffer's non-ghost contents are undefined
 * afterwards.  Bit-identical to `levels` sbp_iterate calls.  stamps: device
 * array of sbp_fused_stamp_words(g) uint32, zero-filled once; epoch: a
 * non-zero value never used before with this stamps array.  Band potentials,
 * Ms >= 32, compiled radius R in {1..4, 7, 8}; otherwise SBP_EUNSUPPORTED. */
SBP_API int sbp_fused_stamp_words(const sbp_grid *g);
SBP_API int sbp_iterate_fused(const sbp_grid *g, const sbp_potential *pot, const float *values,
                              float *msgs_a, float *msgs_b, int levels, int iteration,
                              int flags, unsigned *stamps, unsigned epoch, int lag, int rounds,
                              unsigned long long *err, void *stream);

/* One canonical SEQUENTIAL sweep in place (the reference's default schedule,
 * bp.py:492-503 -> numba_kernels.py:274-407): passes L->R, R->L, T->B, B->T,
 * each a set of independent row / column chains updated in order.  Full grid.
 * Failures: err = min(sweep << 40 | pass << 38 |
 * line * line_len + position), i.e. the reference's first failing message.
 * Band potentials run the chain kernels; ELL / per-edge / dense potentials a
 * warp-per-chain ELL kernel. */
SBP_API int sbp_sweep(const sbp_grid *g, const sbp_potential *pot, const float *values,
                      float *msgs, int sweep, unsigned long long *err, void *stream);

/* sbp_sweep with the fused convergence test (see sbp_iterate_delta): each
 * message written in place is compared with the value it overwrites. */
SBP_API int sbp_sweep_delta(const sbp_grid *g, const sbp_potential *pot, const float *values,
                            float *msgs, int sweep, unsigned long long *err, float *delta,
                            void *stream);

/* Name of the kernel instantiation sbp_iterate (sequential = 0), sbp_sweep
 * (sequential = 1) or sbp_iterate_fused (sequential = 2; falls back to the
 * sbp_iterate name when no fused kernel exists) would launch. */
SBP_API int sbp_plan_name(const sbp_grid *g, const sbp_potential *pot, int sequential,
                          char *buf, int len);

/* Per-node beliefs (sum: normalised product, max: max-normalised scores),
 * normalisers Z (sum only, f64) and argmax labels (lowest index on ties).
 * Any of beliefs / normalizers / labels may be NULL.  bad_node receives
 * min node id whose belief mass is zero (sum), untouched otherwise. */
SBP_API int sbp_beliefs(const sbp_grid *g, int domain, const float *values, const float *msgs,
                float *beliefs, double *normalizers, int32_t *labels,
                unsigned long long *bad_node, void *stream);

/* (2E, M) f32 store in reference directed-edge order (full grid only). */
SBP_API int sbp_gather_store(const sbp_grid *g, const float *msgs, float *out, void *stream);

/* max |a - b| over the real rows of two message buffers -> *out (device f32). */
SBP_API int sbp_max_abs_diff(const sbp_grid *g, const float *a, const float *b, float *out,
                     void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SBP_H */
