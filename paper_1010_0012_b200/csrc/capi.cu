// extern "C" entry points of libsbp.so (declared in include/sbp.h).
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "aux_kernels.cuh"
#include "band_kernel.cuh"
#include "fused_kernel.cuh"
#include "tap_kernel.cuh"

namespace sbp {
template <int MS, int DOM>
BandLaunchFn pick_band_dom(int vl, int R, int rolled);
template <int MS>
BandLaunchFn pick_band(int dom, int vl, int R, int rolled) {
    return dom == SBP_SUM ? pick_band_dom<MS, SBP_SUM>(vl, R, rolled)
                          : pick_band_dom<MS, SBP_MAX>(vl, R, rolled);
}
}

namespace sbp {
template <int MS, int DOM>
BandLaunchFn pick_chain(int R, int vl);
// instantiated in band_ms*_*.cu (keeps this file from compiling every kernel)
#define SBP_EXTERN(MSV)                                                          \
    extern template BandLaunchFn pick_band_dom<MSV, SBP_SUM>(int, int, int);      \
    extern template BandLaunchFn pick_band_dom<MSV, SBP_MAX>(int, int, int);      \
    extern template FusedLaunchFn pick_fused<MSV, SBP_SUM>(int, bool);           \
    extern template FusedLaunchFn pick_fused<MSV, SBP_MAX>(int, bool);
SBP_EXTERN(8) SBP_EXTERN(16) SBP_EXTERN(32) SBP_EXTERN(64) SBP_EXTERN(128) SBP_EXTERN(256)
#undef SBP_EXTERN
#define SBP_EXTERN_TAP(MSV)                                                                  \
    extern template BandLaunchFn pick_band_tap<MSV, SBP_SUM>(int, int, int, int);           \
    extern template BandLaunchFn pick_band_tap<MSV, SBP_MAX>(int, int, int, int);
SBP_EXTERN_TAP(64) SBP_EXTERN_TAP(128) SBP_EXTERN_TAP(256)
#undef SBP_EXTERN_TAP
}

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

// libsbp links its own (static) CUDA runtime, whose per-thread current device
// is independent of the one torch sets.  Every launching entry point
// therefore selects the device that owns its buffers first; otherwise rank k
// of a multi-GPU run would launch on device 0 with device k's pointers.
// sbp_grid::device names it (no driver query per launch); SBP_DEVICE_AUTO
// falls back to looking it up from a buffer pointer.
int select_device_of(const void *p);
int select_device(const sbp_grid *g, const void *p) {
    if (g->device < 0) return select_device_of(p);
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != g->device) cudaSetDevice(g->device);
    return g->device;
}

int select_device_of(const void *p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged) return -1;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != attr.device) cudaSetDevice(attr.device);
    return attr.device;
}

int cuda_status(cudaError_t e, const char *where) {
    if (e == cudaSuccess) return SBP_OK;
    return fail(SBP_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

int check_grid(const sbp_grid *g) {
    if (!g) return fail(SBP_EINVAL, "grid is NULL");
    if (g->H < 1 || g->W < 1 || g->M < 1) return fail(SBP_EINVAL, "bad grid %dx%d M=%d", g->H, g->W, g->M);
    if (g->Ms < g->M || g->Ms % 8) return fail(SBP_EINVAL, "bad padded stride Ms=%d for M=%d", g->Ms, g->M);
    if (g->Ms > 256) return fail(SBP_EUNSUPPORTED, "M=%d > 256 labels is not supported", g->M);
    if (g->rows < 1 || g->r0 < 0 || g->r0 + g->rows > g->H)
        return fail(SBP_EINVAL, "bad strip r0=%d rows=%d of H=%d", g->r0, g->rows, g->H);
    return SBP_OK;
}

const int kRadii[] = {1, 2, 3, 4, 7, 8, 16, 32};   // = SBP_BAND_RADII (band_kernel.cuh)

// Band kernel variant choice, from the B200 A/B runs (tools/ab_vl.sh,
// tools/ab_staged.sh; profiles/r01_kernel_variants.md).  Environment
// overrides: SBP_BAND_VL=8|16, SBP_STAGED=0|1, SBP_ROLL_MIN_R=<r>.
int env_int_raw(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

// The knobs are read once per process (no getenv on the launch path).
struct EnvKnobs {
    int roll_min_r = env_int_raw("SBP_ROLL_MIN_R", -1);
    int staged = env_int_raw("SBP_STAGED", -1);
    int band_vl = env_int_raw("SBP_BAND_VL", 0);
    int fuse_rolled = env_int_raw("SBP_FUSE_ROLLED", 1);
    int chain_vl = env_int_raw("SBP_CHAIN_VL", 8);
    int tap = env_int_raw("SBP_TAP", -1);            // shared-memory-tap kernels: 0 off, 1 on
    int tap_vl = env_int_raw("SBP_TAP_VL", 0);
    int tap_staged = env_int_raw("SBP_TAP_STAGED", -1);
    int tap_rolled = env_int_raw("SBP_TAP_ROLLED", -1);
    int max_blocks = env_int_raw("SBP_MAX_BLOCKS", 0);
    int dense_tc = env_int_raw("SBP_DENSE_TC", 1);   // dense sum-product on the tensor cores: 1 3xTF32,
                                                      // 2 bf16 correction products (faster, 5.7e-6), 0 SIMT
    int tap_lift = env_int_raw("SBP_TAP_LIFT", 1);   // sum, Ms >= 128: R = 5..7 bands run on the R = 8 tap kernel
};
EnvKnobs &knobs() {
    static EnvKnobs k;
    return k;
}
int env_int(const char *name, int dflt) {
    const EnvKnobs &k = knobs();
    int v = -1;
    if (!strcmp(name, "SBP_ROLL_MIN_R")) v = k.roll_min_r;
    else if (!strcmp(name, "SBP_STAGED")) v = k.staged;
    else if (!strcmp(name, "SBP_BAND_VL")) return k.band_vl;
    else if (!strcmp(name, "SBP_FUSE_ROLLED")) return k.fuse_rolled;
    else if (!strcmp(name, "SBP_CHAIN_VL")) return k.chain_vl;
    else return env_int_raw(name, dflt);
    return v < 0 ? dflt : v;
}

// Compiled radius a band of radius R runs on in the synchronous kernels (0:
// none).  Sum-product bands of radius 5..7 at Ms >= 128 (C4: R = 7) are padded
// to 8 with zero taps -- exact no-ops -- so the shared-memory-tap kernel
// (R in {8, 16, 32}) applies: C4 2.27 vs 2.38 ms cold, 2.37 vs 2.46 sustained
// (profiles/r02_ab_c4_tap.txt).  SBP_TAP_LIFT=0 or SBP_TAP=0 keeps R = 7.
int kernel_radius(int Ms, int R, int domain);

struct BandChoice {
    int vl;       // labels per lane
    int variant;  // 0 unrolled, 1 rolled (symmetric, R >= 24), 2 TMA-staged (R <= 16),
                  // 3 shared-memory taps (tap_kernel.cuh; R in {8, 16, 32}, Ms >= 64)
    int rolled = 0, staged = 0;   // variant 3 only
};

// Shared-memory-tap kernels for wide bands (tap_kernel.cuh).  Defaults from
// the B200 A/B (profiles/r02_ab_tap.md; ms per C5 iteration, shuffle kernel ->
// tap kernel): R = 8 sum 1.625 -> 1.520 (v1, VL = 16), max 2.202 -> 2.052
// (v2); R = 16 sum 2.046 -> 1.862, max 3.172 -> 2.778 (v2); R = 32 sum
// 3.091 -> 2.831 (v2), max 4.816 -> 3.893 (v2 rolled: the unrolled four-copy
// body overflows the instruction cache).  Knobs: SBP_TAP=0|1, SBP_TAP_VL,
// SBP_TAP_STAGED (0..3, see below), SBP_TAP_ROLLED.
bool tap_choice(int Ms, int domain, int Rk, bool sym, BandChoice &c) {
    const EnvKnobs &k = knobs();
    const bool compiled = Ms >= 64 && (Rk == 8 || Rk == 16 || Rk == 32);
    // default on where measured faster: every compiled wide band, and R = 8
    // for sum-product at Ms >= 128 (v1, VL = 16: C4 and C5 T=9); max-sum R = 8
    // at Ms < 256 keeps the staged shuffle kernel (not measured)
    const int dflt = (Rk >= 16 || Ms >= 256 || (domain == SBP_SUM && Ms >= 128)) ? 1 : 0;
    if (!compiled || (k.tap < 0 ? dflt : k.tap) == 0) return false;
    c.variant = 3;
    const bool v1_16 = domain == SBP_SUM && Ms >= 128 && Rk == 8;
    c.vl = k.tap_vl == 8 || (k.tap_vl == 16 && domain == SBP_SUM && Ms >= 128) ? k.tap_vl
                                                                               : (v1_16 ? 16 : 8);
    // rolled: 0 four band copies, 1 one copy in a direction loop (symmetric
    // potentials), 2 two copies in a loop of two (v2 only, symmetric)
    c.rolled = k.tap_rolled >= 0 ? (sym ? k.tap_rolled : 0)
                                 : (sym && Rk >= 32 && domain == SBP_MAX ? 1 : 0);
    // staged: 0 register-loaded inputs, 1 TMA-staged inputs, 2 register-light
    // v2 (all four exclusion vectors in shared-memory rows), 3 v2 with the next
    // group's inputs TMA-prefetched into shared memory, 4 v2 with them
    // prefetched into L2, 5 v2 with them double-buffered in registers; 1..5
    // need VL = 8
    c.staged = k.tap_staged >= 0 ? (c.vl == 8 ? k.tap_staged : 0) : (c.vl == 8 ? 2 : 0);
    return true;
}

int band_roll_min_r() {
    return env_int("SBP_ROLL_MIN_R", 24);   // rolled wins at R = 32, loses at R <= 16
}

BandChoice band_choice(int Ms, int domain, int Rk, bool sym) {
    BandChoice c;
    if (tap_choice(Ms, domain, Rk, sym, c)) return c;
    // packed-FP32 build, B200 A/B (profiles/r01_ab_packed.txt): the rolled
    // VL=16 kernel is the fastest for C4 (sum, Ms=128, R=7) cold and
    // sustained; rolled instantiations exist for R in {4, 7, 8} and R >= 24
    // (and for C5 T=9, sum, Ms=256, R=8: 1.51 vs 1.69 ms, r01_ab_rolled_more.txt;
    // at Ms=256 R=4 the staged kernel stays faster, max-sum never rolls)
    const bool rolled_c4 = sym && domain == SBP_SUM &&
                           ((Ms == 128 && (Rk == 4 || Rk == 7 || Rk == 8)) ||
                            (Ms == 256 && (Rk == 7 || Rk == 8)));
    if ((sym && Rk >= band_roll_min_r()) || (rolled_c4 && env_int("SBP_ROLL_MIN_R", 0) != 99)) {
        c.vl = (domain == SBP_SUM && Ms >= 128) ? 16 : 8;
        c.variant = 1;
    } else {
        // Defaults from the B200 A/B (profiles/r01_ab_sustained_3.txt,
        // r01_ab_staged_3.txt; kernel ms per iteration):
        //   max-sum, any Ms         staged VL=8   (C3 0.355 vs 0.372)
        //   sum, Ms=128, R <= 8     plain VL=16   (C4 2.21 cold / 2.43 sustained
        //                                          vs 2.30 / 2.56 plain VL=8)
        //   sum, Ms=256, R <= 4     staged VL=16  (C5 T=5 1.50 vs 1.56)
        //   sum, Ms=256, R 5..8     plain VL=16   (C5 T=9 1.54 vs 1.65)
        //   sum, Ms >= 128, R > 8   staged VL=8   (C5 T=17 2.35 vs 2.44)
        //   sum, Ms < 128           plain VL=8    (C2: variants within noise)
        const bool wide = domain == SBP_SUM && Ms >= 128;
        int staged_default = 0;
        if (domain == SBP_MAX || (wide && Rk > 8)) staged_default = 1;
        else if (wide && Ms >= 256 && Rk <= 4) staged_default = 2;
        // SBP_STAGED: 0 register-loaded, 1 staged VL=8 (2 buffers), 2 staged VL=16
        // (1 buffer; sum, Ms >= 128)
        int staged = env_int("SBP_STAGED", staged_default);
        if (Rk > 16) staged = 0;
        if (staged == 2 && !(domain == SBP_SUM && Ms >= 128)) staged = 1;
        c.variant = staged ? 2 : 0;
        c.vl = staged == 1 ? 8 : (staged == 2 ? 16
                                  : ((wide && Rk <= 8) ? 16 : 8));
    }
    const int v = env_int("SBP_BAND_VL", 0);
    if (v == 8 || (v == 16 && domain == SBP_SUM && Ms >= 128)) c.vl = v;
    return c;
}

sbp::BandLaunchFn band_fn(int Ms, int dom, int vl, int R, int rolled);

// The launch function actually used: the chosen variant if compiled, else
// the always-compiled register-loaded VL=8 kernel (ch is updated to match).
sbp::BandLaunchFn tap_fn(int Ms, int dom, int vl, int R, int rolled, int staged) {
    switch (Ms) {
    case 64: return dom == SBP_SUM ? sbp::pick_band_tap<64, SBP_SUM>(vl, R, rolled, staged)
                                   : sbp::pick_band_tap<64, SBP_MAX>(vl, R, rolled, staged);
    case 128: return dom == SBP_SUM ? sbp::pick_band_tap<128, SBP_SUM>(vl, R, rolled, staged)
                                    : sbp::pick_band_tap<128, SBP_MAX>(vl, R, rolled, staged);
    case 256: return dom == SBP_SUM ? sbp::pick_band_tap<256, SBP_SUM>(vl, R, rolled, staged)
                                    : sbp::pick_band_tap<256, SBP_MAX>(vl, R, rolled, staged);
    default: return nullptr;
    }
}

sbp::BandLaunchFn band_resolve(int Ms, int dom, int Rk, BandChoice &ch) {
    sbp::BandLaunchFn fn = ch.variant == 3 ? tap_fn(Ms, dom, ch.vl, Rk, ch.rolled, ch.staged)
                                           : band_fn(Ms, dom, ch.vl, Rk, ch.variant);
    if (!fn) {
        ch.vl = 8;
        ch.variant = 0;
        fn = band_fn(Ms, dom, 8, Rk, 0);
    }
    return fn;
}

bool band_symmetric(const sbp_potential *pot) {
    bool sym = pot->fbar[0] == pot->fbar[1];
    for (int k = 0; k < 2 * pot->R + 1 && sym; ++k)
        sym = pot->band_w[0][k] == pot->band_w[1][k] ||
              (pot->band_w[0][k] != pot->band_w[0][k] && pot->band_w[1][k] != pot->band_w[1][k]);
    return sym;
}

sbp::BandLaunchFn band_fn(int Ms, int dom, int vl, int R, int rolled) {
    switch (Ms) {
    case 8: return sbp::pick_band<8>(dom, vl, R, rolled);
    case 16: return sbp::pick_band<16>(dom, vl, R, rolled);
    case 32: return sbp::pick_band<32>(dom, vl, R, rolled);
    case 64: return sbp::pick_band<64>(dom, vl, R, rolled);
    case 128: return sbp::pick_band<128>(dom, vl, R, rolled);
    case 256: return sbp::pick_band<256>(dom, vl, R, rolled);
    default: return nullptr;
    }
}

// Geometry and band weights (compiled radius Rk) of a band launch.
void band_args(const sbp_grid *g, const sbp_potential *pot, int Rk, const float *values,
               sbp::BandArgs *a) {
    memset(a, 0, sizeof *a);
    a->values = values;
    a->slot_stride = (long long)(g->rows + 2) * g->W * g->Ms;
    a->H = g->H; a->W = g->W; a->M = g->M; a->Ms = g->Ms; a->r0 = g->r0;
    a->floor_term = pot->floor_term;
    const float pad = pot->domain == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    for (int o = 0; o < 2; ++o) {
        a->fbar[o] = pot->fbar[o];
        for (int k = 0; k < 2 * SBP_MAX_R + 1; ++k) a->w[o][k] = pad;
        for (int d = -pot->R; d <= pot->R; ++d) a->w[o][d + Rk] = pot->band_w[o][d + pot->R];
    }
    sbp::band_pairs(*a, Rk, pad);
}

int kernel_radius(int Ms, int R, int domain) {
    if (knobs().tap_lift && knobs().tap != 0 && domain == SBP_SUM && R >= 5 && R < 8 && Ms >= 128)
        return 8;
    for (int r : kRadii)
        if (r >= R && r < Ms) return r;
    return 0;
}

// The dense sum-product update runs as a 3xTF32 GEMM on the tensor cores
// (dense_tc_kernel.cu) when the table is symmetric -- the caller passes the
// SAME device pointer for both orientations -- and Ms is 128 or 256.
bool dense_on_tensor_cores(const sbp_grid *g, const sbp_potential *pot) {
    return knobs().dense_tc != 0 && pot->domain == SBP_SUM && pot->n_pot == 0 &&
           pot->dense_t[0] && pot->dense_t[0] == pot->dense_t[1] && sbp::dense_tc_supported(g->Ms) &&
           (long long)g->rows * g->W < (1ll << 31);
}

int band_radius(const sbp_grid *g, const sbp_potential *pot) {
    for (int r : kRadii)
        if (r >= pot->R && r < g->Ms) return r;
    return 0;
}

sbp::FusedLaunchFn fused_fn(int Ms, int dom, int R, bool rolled) {
#define SBP_F(MSV)                                                                        \
    case MSV:                                                                             \
        return dom == SBP_SUM ? sbp::pick_fused<MSV, SBP_SUM>(R, rolled)                   \
                              : sbp::pick_fused<MSV, SBP_MAX>(R, rolled);
    switch (Ms) { SBP_F(8) SBP_F(16) SBP_F(32) SBP_F(64) SBP_F(128) SBP_F(256) default: return nullptr; }
#undef SBP_F
}

// Rolled fused body: symmetric band with a compiled rolled instantiation
// (SBP_FUSE_ROLLED=0 forces the unrolled one).
bool fused_rolled(const sbp_grid *g, const sbp_potential *pot, int Rk) {
    (void)g;
    return (Rk == 4 || Rk == 7 || Rk == 8) && band_symmetric(pot) &&
           env_int("SBP_FUSE_ROLLED", 1) != 0;
}

int ell_args(const sbp_grid *g, const sbp_potential *pot, sbp::EllArgs *a) {
    memset(a, 0, sizeof *a);
    if (pot->m_max < 1 || !pot->ell_idx[0] || !pot->ell_w[0])
        return fail(SBP_EINVAL, "ELL potential arrays missing");
    const long long ps = (long long)pot->m_max * g->Ms;
    if (pot->n_pot == 0) {
        if (pot->ell_idx[1] != pot->ell_idx[0] + ps || pot->ell_w[1] != pot->ell_w[0] + ps)
            return fail(SBP_EINVAL, "ELL orientation 1 must follow orientation 0 contiguously");
    } else if (!pot->fbar_all || !pot->pid_h || !pot->pid_v) {
        return fail(SBP_EINVAL, "per-edge ELL potential needs fbar_all, pid_h and pid_v");
    }
    a->slot_stride = (long long)(g->rows + 2) * g->W * g->Ms;
    a->H = g->H; a->W = g->W; a->M = g->M; a->Ms = g->Ms; a->r0 = g->r0;
    a->floor_term = pot->kind == SBP_POT_DENSE ? 0 : pot->floor_term;
    a->m_max = pot->m_max;
    a->fbar[0] = pot->fbar[0];
    a->fbar[1] = pot->fbar[1];
    a->idx = pot->ell_idx[0];
    a->w = pot->ell_w[0];
    a->pot_stride = ps;
    if (pot->n_pot > 0) {
        a->fbar_all = pot->fbar_all;
        a->pid_h = pot->pid_h;
        a->pid_v = pot->pid_v;
    }
    if (pot->accumulate == SBP_ACC_F64) {
        if (pot->domain != SBP_SUM || pot->kind != SBP_POT_ELL || pot->n_pot != 0)
            return fail(SBP_EUNSUPPORTED,
                        "f64 accumulation needs a shared sum-product potential in ELL form");
        if (!pot->ell_w_lo[0] || pot->ell_w_lo[1] != pot->ell_w_lo[0] + ps)
            return fail(SBP_EINVAL, "f64 accumulation needs the low weight plane ell_w_lo");
        a->acc64 = 1;
        a->fbar64[0] = pot->fbar64[0];
        a->fbar64[1] = pot->fbar64[1];
        a->w_lo = pot->ell_w_lo[0];
    } else if (pot->accumulate != SBP_ACC_F32) {
        return fail(SBP_EINVAL, "bad accumulate %d", pot->accumulate);
    }
    return SBP_OK;
}

}  // namespace

namespace sbp {
int launch_block_cap() { return knobs().max_blocks; }
}

extern "C" {

int sbp_version(void) { return 1; }

const char *sbp_last_error(void) { return g_err; }

int sbp_reload_config(void) {
    knobs() = EnvKnobs();
    return SBP_OK;
}

int sbp_band_radius(int Ms, int R) {
    if (R < 0 || R > SBP_MAX_R) return 0;
    for (int r : kRadii)
        if (r >= R && r < Ms) return r;
    return 0;
}

int sbp_padded_labels(int M) {
    if (M < 1) return fail(SBP_EINVAL, "M must be >= 1");
    int ms = 8;
    while (ms < M && ms < 256) ms <<= 1;
    if (ms < M) ms = (M + 7) / 8 * 8;
    return ms;
}

int sbp_init_msgs(const sbp_grid *g, int domain, int ghosts_only, float *msgs, void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (!msgs) return fail(SBP_EINVAL, "msgs is NULL");
    select_device(g, msgs);
    return cuda_status(sbp::launch_init_msgs(msgs, g->H, g->W, g->M, g->Ms, g->r0, g->rows,
                                             domain, ghosts_only ? 1 : 0, (cudaStream_t)stream),
                       "sbp_init_msgs");
}

int sbp_load_values(const sbp_grid *g, int domain, const double *src, float *dst, void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (!src || !dst) return fail(SBP_EINVAL, "NULL pointer");
    select_device(g, dst);
    return cuda_status(sbp::launch_load_values(src, dst, (long long)g->rows * g->W, g->M, g->Ms,
                                               domain, (cudaStream_t)stream),
                       "sbp_load_values");
}

int sbp_stereo_values(const sbp_grid *g, int domain, const uint8_t *left, const uint8_t *right,
                      double beta, double T_u, float *dst, void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (!left || !right || !dst) return fail(SBP_EINVAL, "NULL pointer");
    if (!(beta > 0) || !(T_u > 0)) return fail(SBP_EINVAL, "beta and T_u must be > 0");
    select_device(g, dst);
    return cuda_status(sbp::launch_stereo_values(left, right, (long long)g->rows, g->W, g->M,
                                                 g->Ms, beta, T_u, domain, dst,
                                                 (cudaStream_t)stream),
                       "sbp_stereo_values");
}

static int iterate_impl(const sbp_grid *g, const sbp_potential *pot, const float *values,
                        const float *msgs_in, float *msgs_out, int lr_begin, int lr_end,
                        int iteration, int flags, unsigned long long *err, float *delta,
                        void *stream);

int sbp_iterate(const sbp_grid *g, const sbp_potential *pot, const float *values,
                const float *msgs_in, float *msgs_out, int lr_begin, int lr_end, int iteration,
                int flags, unsigned long long *err, void *stream) {
    return iterate_impl(g, pot, values, msgs_in, msgs_out, lr_begin, lr_end, iteration, flags, err,
                        nullptr, stream);
}

int sbp_iterate_delta(const sbp_grid *g, const sbp_potential *pot, const float *values,
                      const float *msgs_in, float *msgs_out, int lr_begin, int lr_end,
                      int iteration, int flags, unsigned long long *err, float *delta,
                      void *stream) {
    if (!delta) return fail(SBP_EINVAL, "delta is NULL");
    return iterate_impl(g, pot, values, msgs_in, msgs_out, lr_begin, lr_end, iteration, flags, err,
                        delta, stream);
}

static int iterate_impl(const sbp_grid *g, const sbp_potential *pot, const float *values,
                        const float *msgs_in, float *msgs_out, int lr_begin, int lr_end,
                        int iteration, int flags, unsigned long long *err, float *delta,
                        void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (!pot || !values || !msgs_in || !msgs_out || !err) return fail(SBP_EINVAL, "NULL pointer");
    if (pot->domain != SBP_SUM && pot->domain != SBP_MAX) return fail(SBP_EINVAL, "bad domain");
    if (lr_begin < 1 || lr_end > g->rows + 1 || lr_begin > lr_end)
        return fail(SBP_EINVAL, "bad row range [%d, %d) of %d rows", lr_begin, lr_end, g->rows);
    if (lr_begin == lr_end) return SBP_OK;
    if (iteration < 0 || iteration >= (1 << 23)) return fail(SBP_EINVAL, "bad iteration index");
    select_device(g, msgs_out);
    const long long slot = (long long)(g->rows + 2) * g->W * g->Ms;
    cudaStream_t s = (cudaStream_t)stream;
    if (pot->kind == SBP_POT_BAND) {
        if (pot->accumulate != SBP_ACC_F32)
            return fail(SBP_EUNSUPPORTED, "band kernels accumulate in f32 (plan ELL for f64)");
        if (pot->R < 0 || pot->R > SBP_MAX_R) return fail(SBP_EINVAL, "band radius %d", pot->R);
        const int Rk = kernel_radius(g->Ms, pot->R, pot->domain);
        BandChoice ch = band_choice(g->Ms, pot->domain, Rk, band_symmetric(pot));
        sbp::BandLaunchFn fn = Rk ? band_resolve(g->Ms, pot->domain, Rk, ch) : nullptr;
        if (!fn)
            return fail(SBP_EUNSUPPORTED, "no band kernel for Ms=%d R=%d", g->Ms, pot->R);
        sbp::BandArgs a;
        band_args(g, pot, Rk, values, &a);
        a.msgs_in = msgs_in;
        a.msgs_out = msgs_out;
        a.err = err;
        a.lr_begin = lr_begin; a.lr_end = lr_end; a.iteration = iteration;
        a.first = (flags & SBP_ITER_FIRST) ? 1 : 0;
        a.delta = delta;
        return cuda_status(fn(a, s), "sbp_iterate(band)");
    }
    if (pot->kind == SBP_POT_DENSE && pot->n_pot == 0 && pot->dense_t[0] && pot->dense_t[1] &&
        g->Ms >= 32) {
        if (pot->accumulate != SBP_ACC_F32)
            return fail(SBP_EUNSUPPORTED, "the dense kernel accumulates in f32");
        if (delta) return fail(SBP_EUNSUPPORTED, "the dense kernel has no fused convergence test");
        sbp::DenseArgs a;
        a.values = values;
        a.msgs_in = msgs_in;
        a.msgs_out = msgs_out;
        a.err = err;
        a.slot_stride = slot;
        a.H = g->H; a.W = g->W; a.M = g->M; a.Ms = g->Ms; a.r0 = g->r0;
        a.lr_begin = lr_begin; a.lr_end = lr_end; a.iteration = iteration;
        a.first = (flags & SBP_ITER_FIRST) ? 1 : 0;
        a.t[0] = pot->dense_t[0];
        a.t[1] = pot->dense_t[1];
        if (dense_on_tensor_cores(g, pot))
            return cuda_status(sbp::launch_dense_tc(a, knobs().dense_tc == 2, s), "sbp_iterate(dense, tensor cores)");
        return cuda_status(sbp::launch_dense(pot->domain, a, s), "sbp_iterate(dense)");
    }
    if (pot->kind == SBP_POT_ELL || pot->kind == SBP_POT_DENSE) {
        sbp::EllArgs a;
        if (int rc = ell_args(g, pot, &a)) return rc;
        a.values = values;
        a.msgs_in = msgs_in;
        a.msgs_out = msgs_out;
        a.err = err;
        a.lr_begin = lr_begin; a.lr_end = lr_end; a.iteration = iteration;
        a.first = (flags & SBP_ITER_FIRST) ? 1 : 0;
        a.delta = delta;
        return cuda_status(sbp::launch_ell(pot->domain, a, s), "sbp_iterate(ell)");
    }
    return fail(SBP_EINVAL, "unknown potential kind %d", pot->kind);
}

int sbp_fused_stamp_words(const sbp_grid *g) {
    if (int rc = check_grid(g)) return rc;
    return sbp::SBP_FUSE_MAX * g->rows * g->W;   // units of >= 1 pixel
}

int sbp_iterate_fused(const sbp_grid *g, const sbp_potential *pot, const float *values,
                      float *msgs_a, float *msgs_b, int levels, int iteration, int flags,
                      unsigned *stamps, unsigned epoch, int lag, int rounds,
                      unsigned long long *err, void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (!pot || !values || !msgs_a || !msgs_b || !stamps || !err)
        return fail(SBP_EINVAL, "NULL pointer");
    if (levels < 1 || levels > sbp::SBP_FUSE_MAX)
        return fail(SBP_EINVAL, "levels must be in [1, %d]", sbp::SBP_FUSE_MAX);
    if (lag < 2 || rounds < 1) return fail(SBP_EINVAL, "lag must be >= 2 and rounds >= 1");
    if (epoch == 0) return fail(SBP_EINVAL, "epoch 0 is the cleared stamp value");
    if (iteration < 0 || iteration + levels > (1 << 23)) return fail(SBP_EINVAL, "bad iteration index");
    if (pot->kind != SBP_POT_BAND || pot->domain != SBP_SUM && pot->domain != SBP_MAX)
        return fail(SBP_EUNSUPPORTED, "fused iterations need a band potential");
    if (pot->R < 0 || pot->R > SBP_MAX_R) return fail(SBP_EINVAL, "band radius %d", pot->R);
    const int Rk = band_radius(g, pot);
    sbp::FusedLaunchFn fn = Rk ? fused_fn(g->Ms, pot->domain, Rk, fused_rolled(g, pot, Rk)) : nullptr;
    if (!fn) return fail(SBP_EUNSUPPORTED, "no fused kernel for Ms=%d R=%d", g->Ms, pot->R);
    select_device(g, msgs_a);
    sbp::BandArgs a;
    band_args(g, pot, Rk, values, &a);
    a.err = err;
    a.lr_begin = 1;
    a.lr_end = g->rows + 1;
    sbp::FusedArgs f;
    memset(&f, 0, sizeof f);
    float *buf[2] = {msgs_a, msgs_b};
    for (int l = 0; l < levels; ++l) {
        f.lev[l].msgs_in = buf[l & 1];
        f.lev[l].msgs_out = buf[(l + 1) & 1];
        f.lev[l].lr_begin = 1;
        f.lev[l].iteration = iteration + l;
        f.lev[l].first = (l == 0 && (flags & SBP_ITER_FIRST)) ? 1 : 0;
    }
    f.stamps = stamps;
    f.epoch = epoch;
    f.T = levels;
    f.D = lag;
    f.rounds = rounds;
    return cuda_status(fn(a, f, (cudaStream_t)stream), "sbp_iterate_fused");
}

static int sweep_impl(const sbp_grid *g, const sbp_potential *pot, const float *values,
                      float *msgs, int sweep, unsigned long long *err, float *delta, void *stream);

int sbp_sweep(const sbp_grid *g, const sbp_potential *pot, const float *values, float *msgs,
              int sweep, unsigned long long *err, void *stream) {
    return sweep_impl(g, pot, values, msgs, sweep, err, nullptr, stream);
}

int sbp_sweep_delta(const sbp_grid *g, const sbp_potential *pot, const float *values, float *msgs,
                    int sweep, unsigned long long *err, float *delta, void *stream) {
    if (!delta) return fail(SBP_EINVAL, "delta is NULL");
    return sweep_impl(g, pot, values, msgs, sweep, err, delta, stream);
}

static int sweep_impl(const sbp_grid *g, const sbp_potential *pot, const float *values,
                      float *msgs, int sweep, unsigned long long *err, float *delta, void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (!pot || !values || !msgs || !err) return fail(SBP_EINVAL, "NULL pointer");
    if (g->r0 != 0 || g->rows != g->H) return fail(SBP_EINVAL, "sequential sweeps need the full grid");
    if (sweep < 0 || sweep >= (1 << 23)) return fail(SBP_EINVAL, "bad sweep index");
    select_device(g, msgs);
    if (pot->kind != SBP_POT_BAND) {
        sbp::EllArgs a;
        if (int rc = ell_args(g, pot, &a)) return rc;
        a.values = values;
        a.msgs_in = msgs;
        a.msgs_out = msgs;
        a.err = err;
        a.lr_begin = 1; a.lr_end = g->H + 1; a.iteration = sweep;
        a.delta = delta;
        return cuda_status(sbp::launch_ell_sweep(pot->domain, a, (cudaStream_t)stream),
                           "sbp_sweep(ell)");
    }
    if (pot->R < 0 || pot->R > SBP_MAX_R) return fail(SBP_EINVAL, "band radius %d", pot->R);
    if (pot->accumulate != SBP_ACC_F32)
        return fail(SBP_EUNSUPPORTED, "band kernels accumulate in f32 (plan ELL for f64)");
    int Rk = 0;
    for (int r : kRadii)
        if (r >= pot->R && r < g->Ms) { Rk = r; break; }
    sbp::BandLaunchFn fn = nullptr;
    // chain lane width: SBP_CHAIN_VL=16 (sum, Ms >= 128, R <= 8) or 8
    const int chain_vl = env_int("SBP_CHAIN_VL", 8);
    if (Rk) {
#define SBP_C(MSV)                                                                          \
    case MSV:                                                                               \
        fn = pot->domain == SBP_SUM ? sbp::pick_chain<MSV, SBP_SUM>(Rk, chain_vl)           \
                                    : sbp::pick_chain<MSV, SBP_MAX>(Rk, chain_vl);          \
        break;
        switch (g->Ms) { SBP_C(8) SBP_C(16) SBP_C(32) SBP_C(64) SBP_C(128) SBP_C(256) default: break; }
#undef SBP_C
    }
    if (!fn) return fail(SBP_EUNSUPPORTED, "no chain kernel for Ms=%d R=%d", g->Ms, pot->R);
    sbp::BandArgs a;
    memset(&a, 0, sizeof a);
    a.values = values;
    a.msgs_in = msgs;
    a.msgs_out = msgs;
    a.err = err;
    a.slot_stride = (long long)(g->rows + 2) * g->W * g->Ms;
    a.H = g->H; a.W = g->W; a.M = g->M; a.Ms = g->Ms; a.r0 = 0;
    a.lr_begin = 1; a.lr_end = g->H + 1; a.iteration = sweep;
    a.floor_term = pot->floor_term;
    const float pad = pot->domain == SBP_SUM ? 0.0f : -__builtin_huge_valf();
    for (int o = 0; o < 2; ++o) {
        a.fbar[o] = pot->fbar[o];
        for (int k = 0; k < 2 * SBP_MAX_R + 1; ++k) a.w[o][k] = pad;
        for (int d = -pot->R; d <= pot->R; ++d) a.w[o][d + Rk] = pot->band_w[o][d + pot->R];
    }
    sbp::band_pairs(a, Rk, pad);
    a.delta = delta;
    return cuda_status(fn(a, (cudaStream_t)stream), "sbp_sweep");
}

int sbp_plan_name(const sbp_grid *g, const sbp_potential *pot, int sequential, char *buf,
                  int len) {
    if (int rc = check_grid(g)) return rc;
    if (!pot || !buf || len < 1) return fail(SBP_EINVAL, "NULL pointer");
    const char *dom = pot->domain == SBP_SUM ? "sum" : "max";
    if (pot->kind == SBP_POT_BAND) {
        // the chain and fused kernels run on the plain compiled radius
        const int Rk = sequential ? band_radius(g, pot) : kernel_radius(g->Ms, pot->R, pot->domain);
        if (sequential == 1) {
            const int cvl = (env_int("SBP_CHAIN_VL", 8) == 16 && pot->domain == SBP_SUM &&
                             g->Ms >= 128 && Rk <= 8) ? 16 : 8;
            snprintf(buf, len, "chain_pass_kernel<%s,VL=%d,LP=%d,R=%d>", dom, cvl, g->Ms / cvl, Rk);
        } else if (sequential == 2 && Rk && fused_fn(g->Ms, pot->domain, Rk, false)) {
            const int vl = (pot->domain == SBP_SUM && g->Ms >= 128 && Rk <= 8) ? 16 : 8;
            snprintf(buf, len, "band_fused_kernel<%s,VL=%d,LP=%d,R=%d%s>", dom, vl, g->Ms / vl, Rk,
                     fused_rolled(g, pot, Rk) ? ",rolled" : "");
        } else {
            BandChoice ch = band_choice(g->Ms, pot->domain, Rk, band_symmetric(pot));
            if (Rk) band_resolve(g->Ms, pot->domain, Rk, ch);
            if (ch.variant == 3)
                snprintf(buf, len, "%s<%s,VL=%d,LP=%d,R=%d%s%s>",
                         ch.staged >= 2 ? "band_iter_tap2_kernel" : "band_iter_tap_kernel", dom,
                         ch.vl, g->Ms / ch.vl, Rk,
                         ch.rolled == 1 ? ",rolled" : ch.rolled == 2 ? ",rolled2" : "",
                         (ch.staged == 1 || ch.staged == 3) ? ",staged"
                         : ch.staged == 4 ? ",l2pf" : ch.staged == 5 ? ",regpf" : "");
            else
                snprintf(buf, len, "%s<%s,VL=%d,LP=%d,R=%d%s>",
                         ch.variant == 2 ? "band_iter_staged_kernel" : "band_iter_kernel", dom,
                         ch.vl, g->Ms / ch.vl, Rk, ch.variant == 1 ? ",rolled" : "");
        }
    } else if (pot->kind == SBP_POT_DENSE && g->Ms >= 32) {
        if (sequential == 0 && dense_on_tensor_cores(g, pot))
            snprintf(buf, len, "dense_tc_kernel<sum,Ms=%d,%s>", g->Ms,
                     knobs().dense_tc == 2 ? "TF32+2xBF16" : "3xTF32");
        else
            snprintf(buf, len, "dense_iter_kernel<%s,Ms=%d>", dom, g->Ms);
    } else {
        snprintf(buf, len, "%s<%s%s>", sequential == 1 ? "ell_chain_kernel" : "ell_iter_kernel", dom,
                 pot->accumulate == SBP_ACC_F64 ? ",f64" : "");
    }
    return SBP_OK;
}

int sbp_beliefs(const sbp_grid *g, int domain, const float *values, const float *msgs,
                float *beliefs, double *normalizers, int32_t *labels,
                unsigned long long *bad_node, void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (!values || !msgs) return fail(SBP_EINVAL, "NULL pointer");
    select_device(g, msgs);
    return cuda_status(sbp::launch_beliefs(domain, values, msgs, g->W, g->M, g->Ms, g->rows,
                                           beliefs, normalizers, labels, bad_node,
                                           (cudaStream_t)stream),
                       "sbp_beliefs");
}

int sbp_gather_store(const sbp_grid *g, const float *msgs, float *out, void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (g->r0 != 0 || g->rows != g->H) return fail(SBP_EINVAL, "gather needs the full grid");
    if (!msgs || !out) return fail(SBP_EINVAL, "NULL pointer");
    select_device(g, msgs);
    return cuda_status(sbp::launch_gather_store(msgs, g->H, g->W, g->M, g->Ms, out,
                                                (cudaStream_t)stream),
                       "sbp_gather_store");
}

int sbp_max_abs_diff(const sbp_grid *g, const float *a, const float *b, float *out,
                     void *stream) {
    if (int rc = check_grid(g)) return rc;
    if (!a || !b || !out) return fail(SBP_EINVAL, "NULL pointer");
    select_device(g, a);
    return cuda_status(sbp::launch_max_abs_diff(a, b, g->W, g->M, g->Ms, g->rows, out,
                                                (cudaStream_t)stream),
                       "sbp_max_abs_diff");
}

}  // extern "C"
