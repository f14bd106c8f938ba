/*
 * sbp_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU f64 restatement of the reference `sparsebp` grid BP arithmetic
 * (arxiv/paper_1010_0012, /root/reference/pkg/src/sparsebp).  It is the
 * parity checker for the CUDA path and the CPU baseline timed by bench.py;
 * nothing in the product package may link or call it.
 *
 * Parity pin: tests/test_oracle_golden.py checks this file bit-for-bit
 * against golden vectors produced by the reference's own numba bodies
 * (tests/golden/make_golden.py).  Compile with -ffp-contract=off so no
 * multiply-add is fused: the reference (numba, fastmath off) performs every
 * operation with a separate IEEE rounding, in exactly the order below.
 *
 * Two schedules:
 *   - synchronous (Jacobi): every directed message of iteration t+1 is a
 *     function of iteration t only.  This is the schedule of the GPU path;
 *     the per-message arithmetic is the reference's _grid_h_*, _fast_*,
 *     _std_*, _pruned_* and _norm_*_store bodies (numba_kernels.py:35-101,
 *     194-227, 248-271) composed over ping-pong buffers.
 *   - sequential (the reference's canonical in-place directional passes,
 *     numba_kernels.py:230-407, bp.py:492-503).
 *
 * Layout of the synchronous entry point (shared with the CUDA path):
 *   unary  [rows][W][M]            rows of this strip, global rows r0..r0+rows-1
 *   msgs   [4][rows+2][W][M]       local row lr <-> global row r0+lr-1; local
 *                                  rows 0 and rows+1 are halo rows.
 *   slot k of node n holds the message INTO n from its neighbour in
 *   direction k: 0 above, 1 left, 2 right, 3 below (numba_kernels.py:12-18).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DOM_SUM 0
#define DOM_MAX 1
#define K_STANDARD 0
#define K_FAST 1
#define K_PRUNED 2

/* One oriented potential (bp.py:466-489 `_grid_setup`): orientation 0 is the
 * stored potential (L->R, T->B passes), orientation 1 its transpose.
 * `weights` are col_residuals (fast sum), col_values (fast max, pruned), and
 * tableT is the dense transposed table for the standard kernel. */
typedef struct {
    double fbar;
    const int64_t *indptr;   /* M+1 */
    const int64_t *indices;  /* nnz */
    const double *weights;   /* nnz */
    const double *tableT;    /* M*M, tableT[xj*M+xi] = f(xi,xj) */
} oracle_pot;

/* ---- update bodies: numba_kernels.py:35-101 ---------------------------- */

static void std_sum(const double *h, const double *tableT, double *out, int M) {
    for (int xj = 0; xj < M; ++xj) {            /* numba_kernels.py:36-41 */
        double acc = 0.0;
        for (int xi = 0; xi < M; ++xi) acc += tableT[(int64_t)xj * M + xi] * h[xi];
        out[xj] = acc;
    }
}

static void fast_sum(const double *h, const oracle_pot *p, double *out, int M) {
    double S = 0.0;                              /* numba_kernels.py:45-54 */
    for (int xi = 0; xi < M; ++xi) S += h[xi];
    double base = p->fbar * S;
    for (int xj = 0; xj < M; ++xj) {
        double acc = base;
        for (int64_t k = p->indptr[xj]; k < p->indptr[xj + 1]; ++k)
            acc += p->weights[k] * h[p->indices[k]];
        out[xj] = acc;
    }
}

static void pruned_sum(const double *h, const oracle_pot *p, double *out, int M) {
    for (int xj = 0; xj < M; ++xj) {             /* numba_kernels.py:58-63 */
        double acc = 0.0;
        for (int64_t k = p->indptr[xj]; k < p->indptr[xj + 1]; ++k)
            acc += p->weights[k] * h[p->indices[k]];
        out[xj] = acc;
    }
}

static void std_max(const double *h, const double *tableT, double *out, int M) {
    for (int xj = 0; xj < M; ++xj) {             /* numba_kernels.py:67-74 */
        double acc = tableT[(int64_t)xj * M] + h[0];
        for (int xi = 1; xi < M; ++xi) {
            double v = tableT[(int64_t)xj * M + xi] + h[xi];
            if (v > acc) acc = v;
        }
        out[xj] = acc;
    }
}

static void fast_max(const double *h, const oracle_pot *p, double *out, int M) {
    double H = h[0];                             /* numba_kernels.py:78-90 */
    for (int xi = 1; xi < M; ++xi) if (h[xi] > H) H = h[xi];
    double floor_branch = p->fbar + H;
    for (int xj = 0; xj < M; ++xj) {
        double acc = floor_branch;
        for (int64_t k = p->indptr[xj]; k < p->indptr[xj + 1]; ++k) {
            double v = p->weights[k] + h[p->indices[k]];
            if (v > acc) acc = v;
        }
        out[xj] = acc;
    }
}

static void pruned_max(const double *h, const oracle_pot *p, double *out, int M) {
    for (int xj = 0; xj < M; ++xj) {             /* numba_kernels.py:94-101 */
        double acc = -INFINITY;
        for (int64_t k = p->indptr[xj]; k < p->indptr[xj + 1]; ++k) {
            double v = p->weights[k] + h[p->indices[k]];
            if (v > acc) acc = v;
        }
        out[xj] = acc;
    }
}

/* numba_kernels.py:248-271 (_norm_sum_store / _norm_max_store) */
static int norm_store(const double *out, double *dst, int M, int domain) {
    if (domain == DOM_SUM) {
        double s = 0.0;
        for (int x = 0; x < M; ++x) s += out[x];
        if (!(s > 0.0) || s == INFINITY) return 0;
        double inv = 1.0 / s;
        for (int x = 0; x < M; ++x) dst[x] = out[x] * inv;
    } else {
        double mx = out[0];
        for (int x = 1; x < M; ++x) if (out[x] > mx) mx = out[x];
        if (!isfinite(mx)) return 0;
        for (int x = 0; x < M; ++x) dst[x] = out[x] - mx;
    }
    return 1;
}

static void apply_kernel(int kernel, int domain, const double *h, const oracle_pot *p,
                         double *out, int M) {
    if (domain == DOM_SUM) {
        if (kernel == K_STANDARD) std_sum(h, p->tableT, out, M);
        else if (kernel == K_FAST) fast_sum(h, p, out, M);
        else pruned_sum(h, p, out, M);
    } else {
        if (kernel == K_STANDARD) std_max(h, p->tableT, out, M);
        else if (kernel == K_FAST) fast_max(h, p, out, M);
        else pruned_max(h, p, out, M);
    }
}

/* _grid_h_sum / _grid_h_max (numba_kernels.py:194-227): unary first, then
 * slots 0,1,2,3 in ascending order, skipping `excl`. */
static void grid_h(const double *g, const double *m[4], int excl, double *h, int M,
                   int domain) {
    for (int x = 0; x < M; ++x) h[x] = g[x];
    for (int k = 0; k < 4; ++k) {
        if (k == excl) continue;
        if (domain == DOM_SUM) for (int x = 0; x < M; ++x) h[x] *= m[k][x];
        else for (int x = 0; x < M; ++x) h[x] += m[k][x];
    }
}

/* Reference directed-edge id (bp.py:113-133 over mrf.py:401-411 edge order). */
static inline int64_t edge_base(int64_t r, int64_t c, int64_t H, int64_t W) {
    return r * (2 * W - 1) + (r < H - 1 ? 2 * c : c);
}
int64_t oracle_directed_edge_id(int64_t H, int64_t W, int64_t r, int64_t c, int dir) {
    switch (dir) {
    case 0: return 2 * edge_base(r, c, H, W);                 /* n -> n+1 */
    case 1: return 2 * edge_base(r, c - 1, H, W) + 1;         /* n -> n-1 */
    case 2: return 2 * (edge_base(r, c, H, W) + (c + 1 < W)); /* n -> n+W */
    default: return 2 * (edge_base(r - 1, c, H, W) + (c + 1 < W)) + 1; /* n -> n-W */
    }
}

/* _grid_step (numba_kernels.py:230-245): excluded slot and written slot. */
static const int DIR_EXCL[4] = {2, 1, 3, 0};
static const int DIR_WSLOT[4] = {1, 2, 0, 3};
static const int DIR_ORIENT[4] = {0, 1, 0, 1};

/* Initial messages (bp.py:587-601): sum -> 1/M on real slots, 1 on ghost
 * slots; max -> 0 everywhere.  Halo rows are filled as real rows. */
void oracle_init_msgs(double *msgs, int H, int W, int M, int r0, int rows, int domain) {
    int64_t R2 = rows + 2;
    int64_t slot = R2 * W * M;
    for (int k = 0; k < 4; ++k)
        for (int64_t lr = 0; lr < R2; ++lr) {
            int64_t r = r0 + lr - 1;
            for (int64_t c = 0; c < W; ++c) {
                double *p = msgs + k * slot + (lr * W + c) * M;
                double v;
                if (domain == DOM_MAX) v = 0.0;
                else {
                    int ghost = (k == 0 && r <= 0) || (k == 1 && c == 0) ||
                                (k == 2 && c == W - 1) || (k == 3 && r >= H - 1);
                    v = ghost ? 1.0 : 1.0 / M;
                }
                for (int x = 0; x < M; ++x) p[x] = v;
            }
        }
}

/* Potential of the message node (r, c) -> direction dir: shared (pid arrays
 * NULL: pots[orientation]) or per edge (pots[2 * pid + orientation], pid_h[n]
 * for edge (n, n+1), pid_v[n] for (n, n+W); reference _GenericEngine opid,
 * bp.py:516-525). */
static const oracle_pot *pot_of(const oracle_pot *pots, const int *pid_h, const int *pid_v,
                                int64_t W, int64_t r, int64_t c, int dir) {
    int64_t pid = 0;
    if (pid_h) {
        int64_t n = r * W + c;
        pid = dir == 0 ? pid_h[n] : dir == 1 ? pid_h[n - 1] : dir == 2 ? pid_v[n] : pid_v[n - W];
    }
    return &pots[2 * pid + DIR_ORIENT[dir]];
}

/* One synchronous iteration over local rows [lr_begin, lr_end).
 * msgs_out must already hold the ghost/identity values (it is never written
 * at ghost slots).  Returns -1, or the smallest reference directed-edge id
 * whose message could not be normalised. */
int64_t oracle_sync_iterate_pe(int H, int W, int M, int r0, int rows, int lr_begin, int lr_end,
                               int domain, int kernel, const double *unary,
                               const double *msgs_in, double *msgs_out, const oracle_pot *pots,
                               const int *pid_h, const int *pid_v, int nthreads) {
    int64_t slot = (int64_t)(rows + 2) * W * M;
    int64_t fail = INT64_MAX;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(min : fail)
    for (int lr = lr_begin; lr < lr_end; ++lr) {
        double *h = (double *)malloc(sizeof(double) * 2 * M);
        double *out = h + M;
        int64_t r = r0 + lr - 1;
        for (int64_t c = 0; c < W; ++c) {
            int64_t ln = (int64_t)lr * W + c;
            const double *g = unary + ((int64_t)(lr - 1) * W + c) * M;
            const double *m[4];
            for (int k = 0; k < 4; ++k) m[k] = msgs_in + k * slot + ln * M;
            for (int dir = 0; dir < 4; ++dir) {
                int exists = dir == 0 ? c + 1 < W : dir == 1 ? c > 0 : dir == 2 ? r + 1 < H : r > 0;
                if (!exists) continue;
                int64_t step = dir == 0 ? 1 : dir == 1 ? -1 : dir == 2 ? W : -W;
                grid_h(g, m, DIR_EXCL[dir], h, M, domain);
                apply_kernel(kernel, domain, h, pot_of(pots, pid_h, pid_v, W, r, c, dir), out, M);
                double *dst = msgs_out + DIR_WSLOT[dir] * slot + (ln + step) * M;
                if (!norm_store(out, dst, M, domain)) {
                    int64_t id = oracle_directed_edge_id(H, W, r, c, dir);
                    if (id < fail) fail = id;
                }
            }
        }
        free(h);
    }
    return fail == INT64_MAX ? -1 : fail;
}

int64_t oracle_sync_iterate(int H, int W, int M, int r0, int rows, int lr_begin, int lr_end,
                            int domain, int kernel, const double *unary,
                            const double *msgs_in, double *msgs_out,
                            const oracle_pot *pot0, const oracle_pot *pot1, int nthreads) {
    oracle_pot pots[2] = {*pot0, *pot1};
    return oracle_sync_iterate_pe(H, W, M, r0, rows, lr_begin, lr_end, domain, kernel, unary,
                                  msgs_in, msgs_out, pots, NULL, NULL, nthreads);
}

/* One canonical sequential sweep (bp.py:492-503 `_run_grid`): passes
 * L->R, R->L, T->B, B->T, each an in-place chain (grid_pass_*,
 * numba_kernels.py:274-407).  msgs4 is the reference (4, N, M) layout without
 * halo rows.  Returns -1 or the failing flat source node; *fail_dir receives
 * the pass direction.  *madds accumulates the reference madd counter. */
int64_t oracle_seq_sweep_pe(int H, int W, int M, int domain, int kernel,
                            const double *values_in, double *msgs4, const oracle_pot *pots,
                            const int *pid_h, const int *pid_v, int *fail_dir, int64_t *madds) {
    int64_t N = (int64_t)H * W;
    double *h = (double *)malloc(sizeof(double) * 2 * M);
    double *out = h + M;
    int64_t ret = -1;
    for (int dir = 0; dir < 4 && ret < 0; ++dir) {
        int64_t n_lines, line_len, line_stride, step, origin;
        if (dir == 0) { n_lines = H; line_len = W - 1; line_stride = W; step = 1; origin = 0; }
        else if (dir == 1) { n_lines = H; line_len = W - 1; line_stride = W; step = -1; origin = W - 1; }
        else if (dir == 2) { n_lines = W; line_len = H - 1; line_stride = 1; step = W; origin = 0; }
        else { n_lines = W; line_len = H - 1; line_stride = 1; step = -W; origin = (int64_t)(H - 1) * W; }
        int64_t done = 0;
        for (int64_t line = 0; line < n_lines && ret < 0; ++line) {
            int64_t base = line * line_stride + origin;
            for (int64_t pos = 0; pos < line_len; ++pos) {
                int64_t src = base + pos * step;
                const double *m[4];
                for (int k = 0; k < 4; ++k) m[k] = msgs4 + k * N * M + src * M;
                const oracle_pot *p = pot_of(pots, pid_h, pid_v, W, src / W, src % W, dir);
                grid_h(values_in + src * M, m, DIR_EXCL[dir], h, M, domain);
                apply_kernel(kernel, domain, h, p, out, M);
                ++done;
                *madds += kernel == K_STANDARD ? (int64_t)M * M
                        : kernel == K_FAST ? p->indptr[M] - p->indptr[0] + 2 * (int64_t)M
                                           : p->indptr[M] - p->indptr[0];
                if (!norm_store(out, msgs4 + DIR_WSLOT[dir] * N * M + (src + step) * M, M,
                                domain)) {
                    ret = src;
                    *fail_dir = dir;
                    break;
                }
            }
        }
        (void)done;
    }
    free(h);
    return ret;
}

int64_t oracle_seq_sweep(int H, int W, int M, int domain, int kernel, const double *values_in,
                         double *msgs4, const oracle_pot *pot0, const oracle_pot *pot1,
                         int *fail_dir, int64_t *madds) {
    oracle_pot pots[2] = {*pot0, *pot1};
    return oracle_seq_sweep_pe(H, W, M, domain, kernel, values_in, msgs4, pots, NULL, NULL,
                               fail_dir, madds);
}

/* max |a-b| over n entries (reference convergence test, bp.py:671-676). */
double oracle_max_abs_diff(const double *a, const double *b, int64_t n) {
    double d = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double v = fabs(a[i] - b[i]);
        if (v > d) d = v;
    }
    return d;
}
