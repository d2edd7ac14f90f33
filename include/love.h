/*
 * love.h -- C ABI of the B200-native LOVE / KISS-GP hot path (arXiv 1803.06058).
 *
 * LOVE ("LanczOs Variance Estimates", §3) caches a rank-k factor of
 *   C = K_UU W_X (W_X^T K_UU W_X + sigma^2 I)^{-1} W_X^T K_UU          (Eq. 8)
 * from k Lanczos steps on K_hat = W_X^T K_UU W_X + sigma^2 I (KISS-GP, Eq. 5) and
 * answers predictive (co)variances in O(k) (Eq. 10) and posterior samples in
 * O(k(t+m)) per sample (Eqs. 11-15).  Algorithm 1 maps onto
 * love_build_cache (lines P:391-399) and love_predict_var / love_predict_covar.
 *
 * Conventions (all entry points):
 *   - Every data pointer is a DEVICE pointer on the current CUDA device unless stated
 *     otherwise.  Every call is stream-ordered on `stream` (a cudaStream_t passed as void*;
 *     NULL = the legacy default stream).
 *   - Matrices are row-major unless stated otherwise; inputs X are fp64 (reading A3: the
 *     cell index floor((x-lo)/h) must be taken in fp64).
 *   - "V" below is the vector precision chosen by love_opts.precision: float for
 *     LOVE_FP32, double for LOVE_FP64.
 *   - Errors are status codes, never exceptions; love_last_error() returns a thread-local
 *     message for the last non-OK status of the calling thread.
 *   - Ownership: the caller owns every buffer it passes in and every output buffer.  The
 *     library copies what it needs during the call and keeps no reference to caller
 *     memory after the call returns.  A love_cache owns all of its device memory until
 *     love_free().
 *   - Thread safety: a built cache is immutable; concurrent queries on different streams
 *     are safe.  Diagnostic counters are updated with device atomics.
 */
#ifndef LOVE_H_
#define LOVE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOVE_ABI_VERSION 4

typedef struct love_cache love_cache;   /* opaque */

typedef enum {
    LOVE_OK = 0,
    LOVE_ERR_ARG = 1,         /* NULL pointer, bad shape, k < 1, sigma^2 <= 0, m_d < 4, d not in 1..3 */
    LOVE_ERR_RANGE = 2,       /* a training point needs a grid node outside [0, m_d-1] (reading A4) */
    LOVE_ERR_NOT_PD = 3,      /* a pivot of the Cholesky of T_k is <= 0 (reading A13) */
    LOVE_ERR_ZERO_PROBE = 4,  /* the Lanczos probe vector is zero */
    LOVE_ERR_CUDA = 5,        /* a CUDA runtime error (message in love_last_error) */
    LOVE_ERR_NCCL = 6,        /* NCCL could not be loaded / initialised / failed */
    LOVE_ERR_OOM = 7,         /* device allocation failed */
    LOVE_ERR_STATE = 8        /* e.g. love_sample on a cache built with k_sample = 0 */
} love_status;

enum { LOVE_FP32 = 0, LOVE_FP64 = 1 };
enum { LOVE_PROBE_Y = 0, LOVE_PROBE_AVGCOL = 1 };
enum { LOVE_PRIOR_SKI = 0, LOVE_PRIOR_EXACT = 1 };

/* Regular (Kronecker) grid of inducing points: u_{d,i} = lo[d] + i*h[d],
 * i = 0..m[d]-1, flat index row-major (last dimension fastest).  d in 1..3, m[d] >= 4. */
typedef struct {
    int32_t d;
    int32_t reserved;
    int64_t m[3];
    double lo[3];
    double h[3];
} love_grid;

/* Product RBF kernel k(x,x') = outputscale * prod_d exp(-(x_d-x'_d)^2 / (2 l_d^2))
 * (reading A6); the grid kernel matrix is K_UU = outputscale * kron_d T(c_d)
 * with Toeplitz columns c_d[i] = exp(-(i h_d)^2/(2 l_d^2)). */
typedef struct {
    double outputscale;
    double lengthscale[3];
} love_rbf;

typedef struct {
    int32_t precision;      /* LOVE_FP32 (V = float, reductions in fp64) | LOVE_FP64 (V = double) */
    int32_t probe;          /* LOVE_PROBE_Y (default: b = y, reading A1) | LOVE_PROBE_AVGCOL (b = (1/m) W_X^T K_UU 1, P:286;
                               mean cache by Eq. 4) */
    int32_t prior;          /* LOVE_PRIOR_SKI (w*^T K_UU w*, default) | LOVE_PRIOR_EXACT (k(x*,x*)) */
    int32_t reorth_passes;  /* classical Gram-Schmidt passes of the full reorthogonalisation:
                               0 => 1 (fp32) / 2 (fp64, CGS2) */
    double breakdown_tol;   /* tau of the breakdown rule (reading A12); 0 => 1e-6 (fp32) / 1e-10 (fp64) */
    int32_t k_sample;       /* k' of the sampling cache; 0 => no sampling cache */
    int32_t lanczos_mode;   /* LOVE_LANCZOS_AUTO (0) | LOVE_LANCZOS_TWO_PASS (1): classical Gram-Schmidt,
                               Q read twice per step | LOVE_LANCZOS_ONE_READ (2, fp32 only): the
                               lagged one-read fused pass (lanczos_fused.cu) | LOVE_LANCZOS_PARTIAL (3,
                               one GPU, fp32): partial reorthogonalisation (SURVEY 8(f)
                               NEXT #1): Simon's omega recurrence estimates q_{j+1}^T q_i from T; one CGS
                               pass runs only when it exceeds reorth_tol (and on the following step).
                               Opt-in: valid far from convergence; near convergence (var << prior)
                               use the default full reorthogonalisation */
    int32_t var_blocks;     /* LOVE_VAR_BLOCKS_AUTO (0): for d <= 2 the build also stores, per cell c, the
                               fp64 block B_c = (K_UU - Rc Rc^T) restricted to the 4^d stencil nodes of c
                               (SURVEY 8(f) NEXT #3b), and love_predict_var returns w*^T B_c w* (the same
                               Eq. 10 value, reassociated: 4^d(4^d+1)/2 doubles read per query instead of
                               4^d rows of Rc, and the cancellation happens in fp64) |
                               LOVE_VAR_BLOCKS_OFF (1): variances from the Rc rows */
    double reorth_tol;      /* LOVE_LANCZOS_PARTIAL only: reorthogonalise when the estimated loss of
                               orthogonality max_i |q_{j+1}^T q_i| exceeds it; 0 => sqrt(eps) of V */
    int32_t cache_fp64;     /* precision == LOVE_FP32 only (SURVEY §8(c) reading A21, DESIGN reading A12b):
                               LOVE_CACHE_FP64_ON: the cache is built in fp64 (Lanczos vectors, CGS2,
                               breakdown tau 1e-10, Rc, the sampling root: the LOVE_FP64 build) while every
                               query / sample OUTPUT stays V = float.
                               LOVE_CACHE_FP64_AUTO (0, default): the fp32 build runs; if its Lanczos breaks
                               down before k (beta_j < 1e-6 ||T||: the problem is converged, var << prior,
                               and fp32 vectors cannot resolve beta_j below ~1e-7 ||T||, so the late
                               directions are round-off), the cache is rebuilt as
                               with LOVE_CACHE_FP64_ON.  Measured at BASELINE config 5: the fp32 build
                               stops at k_eff = 37 with variances up to 6 % off the oracle at the same k;
                               the fp64 cache runs to the oracle's k_eff = 49 and matches it to ~6e-8.
                               LOVE_CACHE_FP64_OFF: the plain fp32 build, whatever k_eff.
                               love_info.cache_precision reports which build the cache holds; with an fp64
                               cache love_ski_mvm / love_kuu_mvm vectors and the RC / S exports are fp64.
                               For precision == LOVE_FP64 only AUTO / OFF are accepted (no effect). */
    int32_t reserved1;
} love_opts;
enum { LOVE_VAR_BLOCKS_AUTO = 0, LOVE_VAR_BLOCKS_OFF = 1 };
enum { LOVE_CACHE_FP64_AUTO = 0, LOVE_CACHE_FP64_ON = 1, LOVE_CACHE_FP64_OFF = 2 };
enum { LOVE_LANCZOS_AUTO = 0, LOVE_LANCZOS_TWO_PASS = 1, LOVE_LANCZOS_ONE_READ = 2, LOVE_LANCZOS_PARTIAL = 3 };

/* Data-parallel sharding of the training points.  Every rank calls
 * love_build_cache with its own X/y shard and identical grid/kernel/sigma^2/k/opts; the
 * returned caches are identical replicas.  nccl_unique_id: 128 bytes (HOST memory) from
 * love_nccl_unique_id on rank 0, broadcast by the caller.  NULL love_dist => one GPU, no
 * collectives.  world == 1 with an id runs the sharded code path with a one-rank
 * communicator (every all-reduce an identity).  The library keeps one communicator per
 * (id, rank, world, device) for the life of the process, so repeated builds with the same id
 * bootstrap NCCL once.  Errors: LOVE_ERR_ARG (rank/world/id inconsistent), LOVE_ERR_NCCL
 * (NCCL missing or failing). */
typedef struct {
    int32_t rank;
    int32_t world;
    const void* nccl_unique_id;
} love_dist;

typedef struct {
    int32_t k_eff;          /* Lanczos steps kept (< k after breakdown, reading A12) */
    int32_t k_pad;          /* row stride of the cache Rc (k_eff rounded up to a multiple of 4) */
    int32_t k_sample_eff;   /* columns of the sampling root S (0 if none) */
    int32_t precision;
    int64_t n_local;        /* training points on this rank */
    int64_t n_global;       /* training points over all ranks */
    int64_t m_total;        /* inducing points */
    int64_t n_items;        /* interpolation work items (cells split into <= 32-point chunks) */
    double b_norm;          /* ||b|| of the probe (global) */
    const double* alpha;    /* HOST, k_eff entries: diagonal of T_k (owned by the cache) */
    const double* beta;     /* HOST, k_eff-1 entries: off-diagonal of T_k */
    int64_t n_negative_var; /* variance queries that returned < 0 (returned raw, reading A20) */
    int64_t n_out_of_range; /* query points outside the grid (NaN returned) */
    int32_t n_reorth_steps; /* Lanczos steps that ran the reorthogonalisation (all but the last one,
                               except in LOVE_LANCZOS_PARTIAL) */
    int32_t cache_precision; /* precision of the cache's factors (Q, Rc, S; LOVE_FP64 when built with
                               opts.cache_fp64); `precision` above is that of the query / sample outputs */
} love_info;

/* ---------------------------------------------------------------------------------------
 * love_build_cache -- Algorithm 1 pre-computation on this rank's shard.
 *   grid, rbf, opts : HOST structs (opts may be NULL => defaults).
 *   sigma2          : observation noise variance sigma^2 > 0.
 *   X               : n_local x d fp64, row-major.  y : n_local fp64.
 *   k               : Lanczos steps, 1 <= k <= 2048 (k > n_global is clamped to n_global).
 *   dist            : HOST struct or NULL.
 *   out             : HOST pointer receiving the new cache.
 * Runs: interpolation indices/weights, cell sort, K_UU setup, k steps
 * of Lanczos with full reorthogonalisation, streamed Cholesky of
 * T_k, the cache Rc = K_UU W_X Q_k L^{-T} (so Rc Rc^T = R^T R'),
 * the mean cache a (Eq. 6), and the sampling root if opts->k_sample > 0.
 * Synchronises `stream` before returning.  Breakdown is not an error (k_eff < k).
 * On error *out is NULL and nothing is leaked. */
love_status love_build_cache(const love_grid* grid, const love_rbf* rbf, double sigma2,
                             const double* X, const double* y, int64_t n_local, int32_t k,
                             const love_opts* opts, const love_dist* dist, void* stream,
                             love_cache** out);

/* ---------------------------------------------------------------------------------------
 * Additive kernel compositions (Eq. 16): k(x, x') = sum_e k_e(x_e, x'_e) with one
 * 1-D SKI component per input dimension.  The interpolation vectors stack the components'
 * 1-D cubic stencils (4 nonzeros each, 4d per point) and K_UU is block diagonal with the
 * components' Toeplitz blocks; Algorithm 1 runs unchanged on these block forms.
 * Component e: grid u_{e,i} = lo + i*h (i < m, 4 <= m <= 1024), RBF
 * outputscale * exp(-r^2 / (2 lengthscale^2)); its inducing points are numbered after those of
 * components 0..e-1 (m_total = sum_e m_e).
 * ------------------------------------------------------------------------------------ */
typedef struct {
    int64_t m;
    double lo;
    double h;
    double lengthscale;
    double outputscale;
} love_axis;
#define LOVE_MAX_ADDITIVE 32

/* love_build_cache for an additive composition of d (1..LOVE_MAX_ADDITIVE) components.
 *   axes : HOST array of d love_axis.  X : n_local x d fp64 row-major (device).  Other
 *   arguments as love_build_cache.  opts->k_sample must be 0 (LOVE_ERR_ARG otherwise) and
 *   opts->var_blocks is ignored (variances come from the Rc rows of the 4d stencil nodes).
 * The cache answers love_predict_var / love_predict_covar / love_kuu_mvm / love_ski_mvm /
 * love_cache_export like a grid cache; training points keep their original order. */
love_status love_build_cache_additive(const love_axis* axes, int32_t d, double sigma2, const double* X,
                                      const double* y, int64_t n_local, int32_t k, const love_opts* opts,
                                      const love_dist* dist, void* stream, love_cache** out);

/* Predictive variances (Eq. 10 with x*_i = x*_j; Alg. 1):
 *   var(x*) = prior(x*) - || Rc^T w_{x*} ||^2,   prior = w*^T K_UU w* (SKI) or k(x*,x*).
 *   Xs       : t x d fp64 (device).  var_out : t values of V (device).
 *   mean_out : NULL or t values of V: mu(x*) = w*^T a (Eq. 6).
 * Asynchronous.  Out-of-range points give NaN and bump n_out_of_range. */
love_status love_predict_var(const love_cache* cache, const double* Xs, int64_t t,
                             void* var_out, void* mean_out, void* stream);

/* Predictive covariances of t pairs (Xa[i], Xb[i]) (Eq. 10):
 *   cov = prior(x_a, x_b) - (Rc^T w_a) . (Rc^T w_b).   cov_out : t values of V. */
love_status love_predict_covar(const love_cache* cache, const double* Xa, const double* Xb,
                               int64_t t, void* cov_out, void* stream);

/* s joint posterior samples at t points (Eq. 11):
 *   F = mu(X*) 1^T + W_{X*}^T S zeta,   S S^T ~= K_UU - R^T R' (Eqs. 13-15).
 *   zeta : NULL (draw N(0,1) with Philox4x32-10 keyed by `seed`, reading A24) or
 *          k_sample_eff x s fp64 column-major (sample j = column j), for shared-draw parity.
 *   out  : t x s values of V, column-major (sample j is contiguous: out[j*t + i]).
 * Arithmetic: the root S is computed in fp64 (reading A16); G = W_{X*}^T S and mu are accumulated
 * in fp64 and rounded to float, and F = mu 1^T + G zeta runs on the FP32 FMA pipes (SURVEY §8(a)
 * a13) for every cache precision: draws from an fp64 cache are accurate to fp32 round-off.
 * Requires a cache built with k_sample > 0 (else LOVE_ERR_STATE). */
love_status love_sample(const love_cache* cache, const double* Xs, int64_t t, int64_t s,
                        uint64_t seed, const double* zeta, void* out, void* stream);

/* Copies diagnostics into *info (HOST).  Synchronises the device to read the counters. */
love_status love_cache_info(const love_cache* cache, love_info* info);

/* Releases every device buffer of the cache.  NULL is a no-op. */
void love_free(love_cache* cache);

/* Thread-local message of the last non-OK status on the calling thread ("" if none). */
const char* love_last_error(void);

/* --------------------------------------------------------------------------------------
 * Operators of the cached model, for unit parity and for users who need them.
 * Vectors are in the caller's ORIGINAL training-point order.
 * ------------------------------------------------------------------------------------ */

/* out = (W_X^T K_UU W_X + sigma^2 I) v on this rank's points (mvm_K_XX, Alg. 1).
 * v, out : n_local values of Vc (the cache precision: V, or double with opts.cache_fp64).
 * Single-rank caches only (else LOVE_ERR_STATE). */
love_status love_ski_mvm(const love_cache* cache, const void* v, void* out, void* stream);

/* out = K_UU u (Toeplitz / Kronecker-of-Toeplitz MVM).  u, out : m_total of Vc. */
love_status love_kuu_mvm(const love_cache* cache, const void* u, void* out, void* stream);

enum {
    LOVE_EXPORT_RC = 0,        /* m_total x k_pad of Vc, row-major: Rc = K_UU W_X Q L^{-T} */
    LOVE_EXPORT_MEAN = 1,      /* m_total fp64: mean cache a */
    LOVE_EXPORT_S = 2,         /* m_total x ks_pad of Vc, row-major: sampling root (ks_pad = k_sample_eff
                                  rounded up to a multiple of 4) */
    LOVE_EXPORT_PERM = 3       /* n_local int32: sorted position -> original point index */
};
/* Copies an internal array into the caller's DEVICE buffer `dst` of `capacity` bytes.
 * *bytes (HOST, may be NULL) receives the size; dst == NULL only queries the size. */
love_status love_cache_export(const love_cache* cache, int32_t what, void* dst,
                              int64_t capacity, int64_t* bytes, void* stream);

/* Writes a fresh 128-byte NCCL unique id into `out` (HOST).  Call on rank 0 only. */
love_status love_nccl_unique_id(void* out);

/* Number of kernels this library has launched since it was loaded (all threads). */
int64_t love_launch_count(void);

/* LOVE_ABI_VERSION of the loaded library. */
int32_t love_abi_version(void);

/* --------------------------------------------------------------------------------------
 * Phase timing (tracing).  When enabled, the library brackets each phase's kernels with
 * CUDA events on the launching stream; love_profile_read synchronises the device,
 * accumulates the elapsed times and returns per-phase totals (ms) and launch-group counts.
 * Process-global, meant for single-threaded benchmarking.
 * ------------------------------------------------------------------------------------ */
enum {
    LOVE_PROF_SETUP = 0,         /* interpolation records, cell sort, items, K_UU setup */
    LOVE_PROF_SCATTER = 1,       /* u = W q (moments + node pull) */
    LOVE_PROF_KUU = 2,           /* z = K_UU u */
    LOVE_PROF_GATHER = 3,        /* r = W^T z + sigma^2 q, alpha */
    LOVE_PROF_REORTH_DOTS = 4,   /* c = Q^T r' */
    LOVE_PROF_REORTH_UPDATE = 5, /* q~ = r' - Q c, beta^2 */
    LOVE_PROF_SCALARS = 6,       /* tridiagonal Cholesky / breakdown bookkeeping, Rc and a streaming */
    LOVE_PROF_FINISH = 7,        /* Rc transpose */
    LOVE_PROF_QUERY = 8,         /* predict_var / predict_covar */
    LOVE_PROF_SAMPLE_CACHE = 9,  /* sampling root */
    LOVE_PROF_SAMPLE = 10,       /* sample draws */
    LOVE_PROF_COMM = 11,         /* NCCL all-reduces */
    LOVE_PROF_FUSED_PASS = 12,   /* one-read pass: lagged update + gather + moments + Gram dots */
    LOVE_PROF_SAMPLE_GEMM = 13,  /* the draw product F = mu 1^T + G zeta alone (inside LOVE_PROF_SAMPLE) */
    LOVE_PROF_N = 14
};
void love_profile_enable(int32_t on);
/* ms_out, calls_out: HOST arrays of LOVE_PROF_N entries (either may be NULL); reset != 0
 * clears the totals after reading. */
love_status love_profile_read(double* ms_out, int64_t* calls_out, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* LOVE_H_ */
