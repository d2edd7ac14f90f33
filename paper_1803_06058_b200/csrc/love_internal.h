// love_internal.h -- the cache object, device state layout and kernel launchers (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/love.h"
#include "common.cuh"

namespace love {

// ---------------------------------------------------------------------------------------
// Grid geometry.  Flat node index is row-major, last dimension fastest.
// ---------------------------------------------------------------------------------------
struct GridDev {
    int d;
    int m[3];
    int stride[3];          // stride[d-1] = 1
    double lo[3], h[3];
    int m_total;
};

// Additive composition (Eq. 16): per component e a 1-D grid and RBF; component e's
// inducing points are nodes off[e] .. off[e] + m[e] - 1 of the stacked set.
constexpr int kMaxAdd = LOVE_MAX_ADDITIVE;
struct AddDev {
    int d;
    int m[kMaxAdd];
    int off[kMaxAdd + 1];          // off[d] = m_total
    double lo[kMaxAdd], h[kMaxAdd], ls[kMaxAdd], s2[kMaxAdd];
    double c4[kMaxAdd][4];         // c_e[0..3] (variance prior)
};

// Which Lanczos column a step kernel works on.  Step kernels read the step index j from
// device memory (so one captured step graph can be replayed k times); the vector they use
// is base + j * ld, scaled by scale[j]; they do nothing once flags[0] (done) is set.
struct StepRef {
    const int* jdev;        // nullptr -> j = 0
    int64_t ld;             // column stride (0 for a single vector)
    const double* scale;    // scale[j] multiplies the stored column
    const int* flags;       // nullptr -> never skip
};
__device__ __forceinline__ int step_j(const StepRef& r) { return r.jdev ? *r.jdev : 0; }
__device__ __forceinline__ bool step_done(const StepRef& r) { return r.flags != nullptr && r.flags[0] != 0; }

// Device-resident Lanczos state (fp64).  The current step's accumulators live at fixed
// addresses (summed into with atomics by the step kernels, all-reduced between kernels on
// several GPUs, so a captured step graph can be replayed) and are cleared once the step's
// scalars are finalised.
struct LanczosState {
    double* alpha_cur;     // [1]        q_j^T A q_j of the current step
    double* beta2_cur;     // [1]        ||q~_{j+1}||^2 of the current step
    double* c_cur;         // [2][crep][cld] reorthogonalisation dots of the current step (passes 0, 1)
    int crep = 1;          // copies of each pass's dots (CTA b adds to copy b % crep: same-address
                           // fp64 atomics serialise in L2; the update sums the copies)
    int cld = 0;           // stride between copies (0: k + 1)
    int64_t c_len = 0;     // doubles of c_cur (cleared once a step's scalars are final)
    // DGKS-gated second CGS pass (fp64, one GPU): nrm2[0] = ||r'||^2 (pass-0 source, summed by
    // the pass-0 dots), nrm2[1] = ||r''||^2 (pass-0 update output); pass 1 runs only when
    // ||r''||^2 < ||r'||^2 / 2 ("twice is enough")
    double* nrm2 = nullptr;
    int dgks = 0;
    double* bnorm2;        // [1]        ||b||^2
    double* qscale;        // [k+1]      1/||q~_j|| (lazy normalisation of Q's columns)
    double* alpha;         // [k]
    double* beta;          // [k]
    double* Ld;            // [k]        L_jj
    double* Ls;            // [k]        L_{j+1,j}
    double* g;             // [k]        L^{-1} e_1
    double* amax_bmax;     // [2]
    int* flags;            // [4]        done, k_eff, notpd, zero_probe
    int* jdev;             // [1]        current step index j
    int* step_ctr;         // [1]        CTAs done in the step's last kernel (advance_step)
    int* hdone = nullptr;  // mapped host memory: set to 1 with flags[0] (done), so the host stops
                           // replaying the step graph without a stream synchronisation
    int chol = 1;          // finalise the Cholesky row of T too (0: sampling Lanczos on M, reading A15)
    // device-terminated step loop (a CUDA graph WHILE node, one GPU): the step's last CTA
    // clears the loop condition once the Lanczos is done or the step index reaches cond_limit;
    // it also counts the steps run inside the loop in flags[6] (launch accounting)
    unsigned long long cond = 0;
    int cond_limit = 0;
    // partial reorthogonalisation (LOVE_LANCZOS_PARTIAL)
    double* omega;         // [3][k+1]   rows j-1, j, j+1 of Simon's estimates omega_{j,i} ~ q_j^T q_i
    int* pro;              // [4]        reorthogonalise this step, force the next, steps reorthogonalised
    double pro_tol, pro_eps;
    // fused (one-read) mode
    double* AB;            // [k][2][k+1] Gram sums A_i = Q~_i^T r~_j, B_i = Q~_i^T Q~_j of pass j
    double* cvec;          // [k+1]      reorthogonalisation coefficients on Q~_i for the next pass
    double* gam;           // [k+1]      coefficients of u~_i in u~_{j+1}
};

// Column i of the streamed cache, Rc[:, i] = (z_i - L_{i,i-1} Rc[:, i-1]) / L_ii and
// a += ||b|| g_i Rc[:, i] (probe y), computed by extra CTAs of the next step's gather
// kernel once the update kernel's last CTA has finalised the scalars of index i
// (single-GPU Lanczos; i = *jdev - 1, z_i in z[i & 1]).
__host__ __device__ __forceinline__ int64_t c_stride(const LanczosState& st, int k) {
    return st.cld > 0 ? st.cld : k + 1;
}

struct RcStream {
    LanczosState st;
    const double* z0;
    const double* z1;
    double* Rc;          // fp64 column-major m x k
    double* a;           // mean cache (probe y)
    int m;
    int mean_y;
};

struct Cache {
    // ---------------- configuration
    GridDev g;
    love_rbf rbf;
    double sigma2 = 0;
    int precision = LOVE_FP32;          // of the cache's factors (LOVE_FP64 with opts.cache_fp64)
    int out_precision = LOVE_FP32;      // of the query / sample outputs (love_opts.precision)
    int probe = LOVE_PROBE_Y, prior = LOVE_PRIOR_SKI, reorth_passes = 1;
    double tol = 0;
    int k_req = 0, k_sample_req = 0;
    int rank = 0, world = 1;
    void* comm = nullptr;               // ncclComm_t
    int device = 0;
    size_t vsize = 4;                   // sizeof(V)

    // ---------------- additive composition (love_build_cache_additive)
    bool additive = false;
    AddDev ad{};
    int* acell = nullptr;                // [d][n] cell per component, original point order
    void* afrac = nullptr;               // V[d][n] fractional offsets
    int* aperm = nullptr;                // [d][n] component-e cell-sorted position -> point
    int* astart = nullptr;               // component e: cell starts at astart + off[e] + e (m_e + 1)
    void* aMc = nullptr;                 // double[4][m_total] per-cell scatter moments

    // ---------------- training points (sorted by flat cell)
    int64_t n = 0, n_global = 0, ldq = 0;
    int64_t n_items = 0;                 // -1: not listed (d = 1 single-GPU path; love_cache_info reads the count)
    const int* range_flag = nullptr;     // build only: device flag of an off-grid training point, checked
                                         // with the Lanczos flags when no earlier synchronisation did
    void* frac[3] = {nullptr, nullptr, nullptr};   // V[n] per dim (sorted order)
    int* perm = nullptr;                 // [n] sorted -> original
    int* pcell = nullptr;                // d <= 2: [ldq + 4] cell of each sorted point (0 past n)
    int* cell_start = nullptr;           // [m_total+1]
    int* cell_item_start = nullptr;      // [m_total+1]
    int* item_cell = nullptr;            // [n_items]
    int* item_start = nullptr;           // [n_items+1]

    // ---------------- K_UU
    double* cols64 = nullptr;            // [sum m_d] Toeplitz first columns (fp64)
    double h_cols64[3][4] = {};          // host copy of c_d[0..3] (variance-query prior)
    int fft_N = 0, fft_N1 = 0, fft_N2 = 0;
    void* lam = nullptr;                 // double[N] eigenvalues * s^2/N in pass-B layout
    void* fft_buf = nullptr;             // double2[N]
    void* tw1 = nullptr;                 // double2 twiddle tables (line FFTs of N1 / small N)
    void* tw2 = nullptr;                 // (line FFTs of N2)
    void* twF = nullptr;                 // exp(-2 pi i k / N), k < N1
    int rfft_N1 = 0, rfft_N2 = 0;        // real-input convolution at N' = N/2 = rfft_N1 * rfft_N2
    void *rtw1 = nullptr, *rtw2 = nullptr, *rtwF = nullptr, *rtwU1 = nullptr, *rtwU2 = nullptr;
    void* rlam = nullptr;                // double[N'+1] lambda * s^2 / N, natural order
    void* ktmp[2] = {nullptr, nullptr};  // double[m] scratch for axis passes
    int ax_N[3] = {0, 0, 0};             // d > 1: per-axis circulant length (0: dense axis product)
    void* ax_tw[3] = {nullptr, nullptr, nullptr};   // exp(-2 pi i k / N_d), k < N_d
    void* ax_lam[3] = {nullptr, nullptr, nullptr};  // double[N_d]: lambda_d / N_d

    // ---------------- Lanczos
    int k_alloc = 0;
    void* Q = nullptr;                   // V[ldq * (k+1)] column-major, unnormalised columns
    void* r = nullptr;                   // V[ldq]
    void* u = nullptr;                   // double[m]
    void* z[2] = {nullptr, nullptr};     // double[m]
    void* M = nullptr;                   // double[4^d * n_items] per-item stencil moments
    void* M2 = nullptr;                  // second moments buffer (fused mode: moments of Q~_j)
    void* Mc = nullptr;                  // d = 1: double[4][m+4] per-cell stencil moments of the scatter
    int64_t cond_nodes = 0;              // kernels per iteration of the device-terminated step loop
    int cond_steps = 1;                  // Lanczos steps per iteration
    void* pullT = nullptr;               // d >= 2: double[4^(d-1)][m] last-axis pull of the scatter
    void* pullV = nullptr;               // d = 3: double[4][m] middle-axis pull
    void* Rc_col = nullptr;              // double[m * k] column-major (build only)
    // fused (one-read) Lanczos mode
    bool fused = false;
    bool partial = false;                // LOVE_LANCZOS_PARTIAL
    int tile_cap = 0;                    // max points per fused-pass tile
    int64_t n_tiles = 0;
    int* tile_first = nullptr;           // [n_tiles+1] first item of each tile
    void* tile_meta = nullptr;           // [n_tiles] per-tile descriptors (lanczos_fused.cu)
    alignas(64) unsigned char qmap[128] = {};   // CUtensorMap of Q~ (lanczos_fused.cu)
    int fused_threads = 256;
    double* U64 = nullptr;               // [3][m] u~_{j-1}, u~_j, u~_{j+1} (rolling, fp64)
    float* U32 = nullptr;                // [k+1][m] every u~_i in fp32 (reorth correction)
    void* Rc = nullptr;                  // V[m * k_pad] row-major
    void* Rc64 = nullptr;                // fp32 caches: double[m * k_pad] row-major, made by the first
                                         // love_predict_covar (covariances from fp64 rows)
    void* a = nullptr;                   // double[m] mean cache
    void* vblk = nullptr;                // d <= 2: double[m][4^d(4^d+1)/2] per-cell variance blocks
    bool var_blocks_off = false;
    void* ysort = nullptr;               // V[ldq] targets in sorted order (probe avg only)
    double* one = nullptr;               // device 1.0 (scale of un-normalised MVMs)
    double* scal = nullptr;              // backing store of LanczosState
    LanczosState st;
    unsigned long long* counters = nullptr;   // [2] negative variances, out-of-range queries

    // ---------------- results
    int k_eff = 0, k_pad = 0;
    int n_reorth_steps = 0;
    int k_sample_eff = 0, ks_pad = 0;
    void* S = nullptr;                   // V[m * ks_pad] row-major sampling root
    double b_norm = 0;
    std::vector<double> h_alpha, h_beta;
    std::vector<double> h_evals;         // eigenvalues of T' (sampling cache)

    std::vector<void*> allocs;           // everything to release
    unsigned long long* trace = nullptr; // LOVE_TRACE: [k][kTraceKernels][start, end] (ns)
    char* slab = nullptr;                // small buffers are carved from zeroed slabs (dalloc)
    size_t slab_used = 0;
};

// ---------------------------------------------------------------------------------------
// Error plumbing
// ---------------------------------------------------------------------------------------
void set_error(const std::string& msg);
struct LoveError {
    love_status status;
    std::string msg;
};
// internal status (never returned through the ABI): the fp32 build broke down before k under
// LOVE_CACHE_FP64_AUTO and must be rebuilt with an fp64 cache (love_api.cu)
constexpr love_status kRebuildFp64 = (love_status)100;
void cuda_check(cudaError_t e, const char* what);
// raises a kernel's dynamic shared-memory limit once (cudaFuncSetAttribute is a host call)
void ensure_smem(const void* fn, size_t bytes);
void* dalloc(Cache& c, size_t bytes, cudaStream_t s);   // zero-filled, owned by the cache
void* pinned_scratch(size_t bytes);                      // this thread's pinned host staging buffer
// owned by the cache, NOT zero-filled: only for buffers every reader finds written first
// (LOVE_POISON=1 fills them with NaN bytes instead, to prove it)
void* dalloc_unset(Cache& c, size_t bytes, cudaStream_t s);

// ---------------------------------------------------------------------------------------
// Launchers (each file defines its own kernels; V = float | double)
// ---------------------------------------------------------------------------------------
// interp.cu
void launch_interp_points(const Cache& c, const double* X, int64_t n, int* cell, double* frac64,
                          int* range_flag, cudaStream_t s);
void launch_counting_sort(Cache& c, const int* cell, const double* frac64, const double* y,
                          int64_t n, void* b_out, cudaStream_t s);   // fills perm, frac, cells
void launch_build_items(Cache& c, cudaStream_t s);                 // after n_items known
int64_t count_items_host(Cache& c, cudaStream_t s);                 // syncs
// keys in [0, nbins): start[nbins+1] = exclusive scan of the histogram, perm[start[k] ..] = the
// indices with key k (order within a key unspecified)
void counting_sort_keys(const int* keys, int64_t n, int nbins, int* start, int* perm, cudaStream_t s);
// ski.cu
// d = 1 (non-fused caches): per-cell moments into c.Mc, then u unless moments_only (the
// K_UU MVM then reads the moments itself, launch_kuu(..., Mc))
template <typename V> void launch_scatter(const Cache& c, const V* qbase, StepRef ref, double* u,
                                          cudaStream_t s, bool moments_only = false);
template <typename V> void launch_gather(const Cache& c, const double* z, const V* qbase, StepRef ref, V* r,
                                         double* alpha_base, cudaStream_t s, const RcStream* rs = nullptr);
// device part of the streamed cache column (RcStream), rows p0, p0+stride, ...
__device__ __forceinline__ void stream_rc_column(const RcStream& rs, int p0, int stride) {
    const int i = *rs.st.jdev - 1;
    const int* fl = rs.st.flags;
    if (i < 0 || fl[1] <= i || fl[2] || fl[3]) return;
    const double ld = rs.st.Ld[i];
    const double lsub = i > 0 ? rs.st.Ls[i - 1] : 0.0;
    const double ag = sqrt(rs.st.bnorm2[0]) * rs.st.g[i];
    const double* __restrict__ z = (i & 1) ? rs.z1 : rs.z0;
    for (int p = p0; p < rs.m; p += stride) {
        const double prev = i > 0 ? rs.Rc[(int64_t)(i - 1) * rs.m + p] : 0.0;
        const double v = (z[p] - lsub * prev) / ld;
        rs.Rc[(int64_t)i * rs.m + p] = v;
        if (rs.mean_y) rs.a[p] += ag * v;
    }
}
template <typename A, typename B> void launch_convert(const A* in, B* out, int64_t n, cudaStream_t s);
void launch_nodepass(const Cache& c, StepRef ref, double* u, cudaStream_t s);   // from c.M
template <typename V> void launch_permute(const Cache& c, const V* in, V* out, bool to_sorted,
                                          cudaStream_t s);
// kuu.cu
void setup_kuu(Cache& c, cudaStream_t s);
// z = K_UU u; for d = 1, u may instead be given as the per-cell moments Mc of launch_scatter
// pull3 (d = 3, fuse_pull3): u is not materialised -- the first axis product forms it from the
// scatter's fp32 last-axis sums (c.pullT) and the step's scale
void launch_kuu(const Cache& c, const double* u, double* z, cudaStream_t s, const double* Mc = nullptr,
                const StepRef* pull3 = nullptr);
bool fuse_pull3(const Cache& c);
// lanczos.cu
void run_lanczos(Cache& c, cudaStream_t s);
// L2 residency of Q~'s first columns for one build (nullptr: not used); end after the build's
// final synchronisation (restores the device's persisting-L2 set-aside)
void* l2_persist_begin(const Cache& c, cudaStream_t s);
void l2_persist_end(void* h);
// Host side of the early stop of step-graph replays (ReplayThrottle in lanczos.cu): a mapped
// host flag the device sets at breakdown, and at most kReplayWindow replays in flight beyond the
// last one the host has seen complete.
struct ReplayThrottle {
    volatile int* h = nullptr;     // host view of the done flag
    int* d = nullptr;              // device view (LanczosState::hdone)
    cudaEvent_t* ev = nullptr;
    explicit ReplayThrottle(int device);
    bool stopped() const { return *h != 0; }
    // before replay i: wait until replay i - kReplayWindow has completed; false once done
    bool admit(int i);
    void launched(int i, cudaStream_t s);
};
void launch_reorth_pass_f64(const LanczosState& st, double* Q, int64_t ldq, int64_t n, int k, int pass,
                            int last_pass, const double* r, double tol, cudaStream_t s);
void launch_init_q0(const LanczosState& st, cudaStream_t s);
void run_lanczos_fused(Cache& c, cudaStream_t s);   // lanczos_fused.cu
void setup_fused(Cache& c, cudaStream_t s);
void finish_cache(Cache& c, cudaStream_t s);    // Rc -> row-major m x k_pad
void launch_rc_rows64(const Cache& c, double* out, cudaStream_t s);   // fp64 row-major Rc (m x k_pad)
// in-pipeline kernel trace (LOVE_TRACE=1, common.cuh): per-translation-unit binders, and the
// build-side driver (trace_begin before the Lanczos replays, trace_report after its sync)
void trace_bind_ski(unsigned long long* p, cudaStream_t s);
void trace_bind_kuu(unsigned long long* p, cudaStream_t s);
void trace_bind_lanczos(unsigned long long* p, cudaStream_t s);
void trace_bind_sample(unsigned long long* p, cudaStream_t s);
void trace_begin(Cache& c, int k, cudaStream_t s);
void trace_end(cudaStream_t s);
void trace_report(Cache& c, int k_eff);
void avgcol_probe(Cache& c, cudaStream_t s);    // Q~[:, 0] = (1/m) W^T K_UU 1   (probe avg)
void mean_cache_eq4(Cache& c, cudaStream_t s);  // a = Rc L^{-1} Q^T y after the Lanczos loop
// query.cu
template <typename V> void launch_predict(const Cache& c, const double* Xa, const double* Xb,
                                          int64_t t, V* out, V* mean_out, cudaStream_t s);
void build_var_blocks(Cache& c, cudaStream_t s);   // per-cell fp64 variance blocks (d <= 2)
// additive.cu
void additive_setup(Cache& c, const double* X, const double* y, int* range_flag, cudaStream_t s);
template <typename V> void add_scatter(const Cache& c, const V* qbase, StepRef ref, double* u, cudaStream_t s);
void add_kuu(const Cache& c, const double* u, double* z, cudaStream_t s);
template <typename V> void add_gather(const Cache& c, const double* z, const V* qbase, StepRef ref, V* r,
                                      double* alpha_base, cudaStream_t s, const RcStream* rs);
template <typename V> void add_predict(const Cache& c, const double* Xa, const double* Xb, int64_t t, V* out,
                                       V* mean_out, cudaStream_t s);
// sample.cu
void build_sampling_cache(Cache& c, cudaStream_t s);
template <typename V> void launch_sample(const Cache& c, const double* Xs, int64_t t, int64_t ns,
                                         uint64_t seed, const double* zeta, V* out,
                                         cudaStream_t s);
// Instantiated step graphs kept across builds (per thread, keyed by purpose + shape): a build
// whose freshly captured graph has the topology of a cached one refreshes it with
// cudaGraphExecUpdate (new buffer pointers) instead of instantiating again.  The returned exec
// is owned by the cache (do not destroy it).
cudaGraphExec_t graph_exec_cached(cudaGraph_t g, const std::string& key);
// host-side timeline of a build (LOVE_HOST_TIMING=1: printed to stderr at the end of the build)
void host_mark(const char* what);
void host_marks_flush();
// profile.cpp (phase timing, love_profile_*)
bool profiling();
void prof_begin(int cat, cudaStream_t s);
void prof_end(int cat, cudaStream_t s);
struct ProfScope {
    int cat;
    cudaStream_t s;
    ProfScope(int c, cudaStream_t st) : cat(c), s(st) { prof_begin(cat, s); }
    ~ProfScope() { prof_end(cat, s); }
};
// nccl_shim.cpp
bool nccl_available(std::string* why);
love_status nccl_get_unique_id(void* out128);
love_status nccl_comm_init(Cache& c, const void* id128);
void nccl_comm_destroy(Cache& c);
void allreduce_sum(const Cache& c, void* buf, int64_t count, bool is_double, cudaStream_t s);
void allreduce_sum_i64(const Cache& c, int64_t* buf, int64_t count, cudaStream_t s);

}  // namespace love
