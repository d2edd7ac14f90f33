// love_api.cu -- the extern "C" boundary (include/love.h) and the build orchestration of
// Algorithm 1's pre-computation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "love_internal.h"

namespace love {

std::atomic<int64_t> g_launch_count{0};
thread_local bool t_pdl = false;
thread_local const int* t_done = nullptr;

namespace {
thread_local std::string t_err;
}

void set_error(const std::string& msg) { t_err = msg; }

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    (void)cudaGetLastError();
    throw LoveError{e == cudaErrorMemoryAllocation ? LOVE_ERR_OOM : LOVE_ERR_CUDA,
                    std::string(what) + ": " + cudaGetErrorString(e)};
}

void ensure_smem(const void* fn, size_t bytes) {
    // the attribute is per device context: cache it per (device, kernel)
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    if (bytes <= 48 * 1024) return;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> g(mu);
    size_t& cur = done[{dev, fn}];
    if (cur >= bytes) return;
    cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), "smem attr");
    cur = bytes;
}

// Buffers up to kSlabPiece bytes are carved (256-byte aligned) from slabs of kSlab bytes that
// are zeroed once when they are allocated: a build's few dozen state buffers cost a handful of
// allocation / memset calls instead of two each (LOVE_NO_SLAB: one allocation per buffer).
constexpr size_t kSlab = size_t(4) << 20, kSlabPiece = size_t(256) << 10;

void* dalloc(Cache& c, size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    bytes = std::max<size_t>(bytes, 16);
    static const bool no_slab = std::getenv("LOVE_NO_SLAB") != nullptr;
    if (!no_slab && bytes <= kSlabPiece) {
        bytes = (bytes + 255) & ~size_t(255);
        if (c.slab == nullptr || c.slab_used + bytes > kSlab) {
            cuda_check(cudaMallocAsync(&p, kSlab, s), "cudaMallocAsync(slab)");
            c.allocs.push_back(p);
            cuda_check(cudaMemsetAsync(p, 0, kSlab, s), "cudaMemsetAsync(slab)");
            c.slab = (char*)p;
            c.slab_used = 0;
        }
        p = c.slab + c.slab_used;
        c.slab_used += bytes;
        return p;
    }
    cuda_check(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
    c.allocs.push_back(p);
    cuda_check(cudaMemsetAsync(p, 0, bytes, s), "cudaMemsetAsync");
    return p;
}

void* dalloc_unset(Cache& c, size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    bytes = std::max<size_t>(bytes, 16);
    cuda_check(cudaMallocAsync(&p, bytes, s), "cudaMallocAsync");
    c.allocs.push_back(p);
    static const bool poison = std::getenv("LOVE_POISON") != nullptr;
    if (poison) cuda_check(cudaMemsetAsync(p, 0xff, bytes, s), "cudaMemsetAsync(poison)");
    return p;
}

void* pinned_scratch(size_t bytes) {
    thread_local void* p = nullptr;
    thread_local size_t cap = 0;
    if (bytes > cap) {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = std::max<size_t>(bytes, 64 << 10);
        cuda_check(cudaHostAlloc(&p, cap, cudaHostAllocDefault), "cudaHostAlloc(scratch)");
    }
    return p;
}

namespace {

void release(Cache* c) {
    if (!c) return;
    for (void* p : c->allocs) cudaFree(p);
    c->allocs.clear();
    nccl_comm_destroy(*c);
    delete c;
}

struct TempPool {                   // stream-ordered temporaries of one call
    cudaStream_t s;
    std::vector<void*> ps;
    explicit TempPool(cudaStream_t st) : s(st) {}
    void* get(size_t bytes) {
        void* p = nullptr;
        cuda_check(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), s), "cudaMallocAsync(tmp)");
        ps.push_back(p);
        return p;
    }
    ~TempPool() {
        for (void* p : ps) cudaFreeAsync(p, s);
    }
};

void keep_pool_memory(int dev) {
    static bool done[64] = {false};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[dev] = true;
}

__global__ void init_state_kernel(int* flags, int k, double* one) {
    if (threadIdx.x == 0) {
        flags[0] = 0;
        flags[1] = k;
        flags[2] = 0;
        flags[3] = 0;
        one[0] = 1.0;
    }
}

// The build runs on a private non-blocking stream (the caller's stream may be the legacy
// default stream, which cannot be captured into a CUDA graph); it is ordered after the
// caller's stream by an event and the build synchronises it before returning.
cudaStream_t work_stream(int dev) {
    thread_local cudaStream_t streams[64] = {nullptr};
    if (dev < 0 || dev >= 64) throw LoveError{LOVE_ERR_CUDA, "device index out of range"};
    if (!streams[dev]) cuda_check(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking), "stream create");
    return streams[dev];
}

void order_after(cudaStream_t waiter, cudaStream_t producer) {
    cudaEvent_t e;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    cuda_check(cudaEventRecord(e, producer), "event record");
    cuda_check(cudaStreamWaitEvent(waiter, e, 0), "stream wait");
    cuda_check(cudaEventDestroy(e), "event destroy");
}

// The exception in flight, as a status (every extern "C" entry point catches everything:
// nothing may unwind through the C ABI).  Host allocation failures map to LOVE_ERR_OOM.
LoveError current_error() {
    try {
        throw;
    } catch (const LoveError& e) {
        return e;
    } catch (const std::bad_alloc&) {
        return LoveError{LOVE_ERR_OOM, "host allocation failed"};
    } catch (const std::exception& e) {
        return LoveError{LOVE_ERR_CUDA, std::string("internal error: ") + e.what()};
    } catch (...) {
        return LoveError{LOVE_ERR_CUDA, "internal error: unknown exception"};
    }
}

// The fp64 row-major copy of an fp32 cache's Rc, made once per cache (under a lock, finished
// before it is published: concurrent queries on other streams never see it half written).
void* rc_rows64(const Cache& cc, cudaStream_t s) {
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    Cache& c = const_cast<Cache&>(cc);
    if (c.Rc64 == nullptr) {
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, sizeof(double) * (size_t)c.g.m_total * std::max(c.k_pad, 4)), "cudaMalloc(Rc64)");
        c.allocs.push_back(p);
        launch_rc_rows64(c, (double*)p, s);
        cuda_check(cudaStreamSynchronize(s), "Rc64 sync");
        c.Rc64 = p;
    }
    return c.Rc64;
}

love_status fail(const LoveError& e) {
    set_error(e.msg);
    return e.status;
}

void validate_build(const love_grid* grid, const love_rbf* rbf, double sigma2, const double* X,
                    const double* y, int64_t n_local, int32_t k, love_cache** out) {
    if (!grid || !rbf || !out) throw LoveError{LOVE_ERR_ARG, "NULL grid/rbf/out"};
    if (grid->d < 1 || grid->d > 3) throw LoveError{LOVE_ERR_ARG, "grid.d must be 1..3"};
    int64_t mt = 1;
    for (int d = 0; d < grid->d; ++d) {
        if (grid->m[d] < 4) throw LoveError{LOVE_ERR_ARG, "grid.m[d] must be >= 4"};
        if (!(grid->h[d] > 0.0) || !std::isfinite(grid->lo[d]))
            throw LoveError{LOVE_ERR_ARG, "grid.h[d] must be > 0 and lo finite"};
        if (!(rbf->lengthscale[d] > 0.0)) throw LoveError{LOVE_ERR_ARG, "lengthscale must be > 0"};
        mt *= grid->m[d];
    }
    if (mt >= (int64_t(1) << 30)) throw LoveError{LOVE_ERR_ARG, "m_total too large"};
    if (!(rbf->outputscale > 0.0)) throw LoveError{LOVE_ERR_ARG, "outputscale must be > 0"};
    if (!(sigma2 > 0.0)) throw LoveError{LOVE_ERR_ARG, "sigma^2 must be > 0"};
    if (k < 1) throw LoveError{LOVE_ERR_ARG, "k must be >= 1"};
    // per-step shared memory holds 8 (k+1) fp64 partial dots (reorthogonalisation)
    if (k > 2048) throw LoveError{LOVE_ERR_ARG, "k must be <= 2048"};
    if (n_local < 0 || n_local >= (int64_t(1) << 31)) throw LoveError{LOVE_ERR_ARG, "bad n_local"};
    if (n_local > 0 && (!X || !y)) throw LoveError{LOVE_ERR_ARG, "NULL X/y"};
}

}  // namespace

}  // namespace love

namespace love {
namespace {

love_opts checked_opts(const love_opts* opts) {
    love_opts o{};
    o.precision = LOVE_FP32;
    if (opts) o = *opts;
    if (o.precision != LOVE_FP32 && o.precision != LOVE_FP64) throw LoveError{LOVE_ERR_ARG, "bad precision"};
    if (o.probe != LOVE_PROBE_Y && o.probe != LOVE_PROBE_AVGCOL) throw LoveError{LOVE_ERR_ARG, "bad probe"};
    if (o.prior != LOVE_PRIOR_SKI && o.prior != LOVE_PRIOR_EXACT) throw LoveError{LOVE_ERR_ARG, "bad prior"};
    if (o.k_sample < 0 || o.reorth_passes < 0) throw LoveError{LOVE_ERR_ARG, "bad opts"};
    if (o.var_blocks != LOVE_VAR_BLOCKS_AUTO && o.var_blocks != LOVE_VAR_BLOCKS_OFF)
        throw LoveError{LOVE_ERR_ARG, "bad var_blocks"};
    if (o.cache_fp64 < LOVE_CACHE_FP64_AUTO || o.cache_fp64 > LOVE_CACHE_FP64_OFF)
        throw LoveError{LOVE_ERR_ARG, "bad cache_fp64"};
    if (o.cache_fp64 == LOVE_CACHE_FP64_ON && o.precision != LOVE_FP32)
        throw LoveError{LOVE_ERR_ARG, "cache_fp64 = LOVE_CACHE_FP64_ON applies to precision == LOVE_FP32 only"};

    return o;
}

// Cache creation and everything both model structures share before the structure-specific
// setup: options, NCCL communicator, global n, k clamp, Q's leading dimension.
Cache* begin_build(const love_opts& o, double sigma2, int64_t n_local, int32_t& k, const love_dist* dist,
                   cudaStream_t s) {
    Cache* c = new Cache();
    try {
        cuda_check(cudaGetDevice(&c->device), "cudaGetDevice");
        keep_pool_memory(c->device);
        c->sigma2 = sigma2;
        // cache_fp64 (reading A12b): the whole build runs as the fp64 build; only the query and
        // sample outputs keep the caller's precision
        const int cprec = o.cache_fp64 == LOVE_CACHE_FP64_ON ? LOVE_FP64 : o.precision;
        c->precision = cprec;
        c->out_precision = o.precision;
        c->vsize = cprec == LOVE_FP64 ? 8 : 4;
        c->probe = o.probe;
        c->prior = o.prior;
        if (o.reorth_passes > 2) throw LoveError{LOVE_ERR_ARG, "reorth_passes must be 0, 1 or 2"};
        c->reorth_passes = o.reorth_passes > 0 ? o.reorth_passes : (cprec == LOVE_FP64 ? 2 : 1);
        int mode = o.lanczos_mode;
        if (const char* e = std::getenv("LOVE_LANCZOS_MODE")) mode = std::atoi(e);
        if (mode < 0 || mode > 3) throw LoveError{LOVE_ERR_ARG, "bad lanczos_mode"};
        if (mode == LOVE_LANCZOS_ONE_READ && cprec != LOVE_FP32)
            throw LoveError{LOVE_ERR_ARG, "the one-read Lanczos pass is fp32 only"};
        c->fused = mode == LOVE_LANCZOS_ONE_READ;
        c->partial = mode == LOVE_LANCZOS_PARTIAL;
        if (c->partial && dist && (dist->world > 1 || dist->nccl_unique_id))
            throw LoveError{LOVE_ERR_ARG, "partial reorthogonalisation runs on one GPU"};
        if (c->partial && cprec != LOVE_FP32)
            throw LoveError{LOVE_ERR_ARG, "partial reorthogonalisation is fp32 only"};
        if (!(o.reorth_tol >= 0.0)) throw LoveError{LOVE_ERR_ARG, "reorth_tol must be >= 0"};
        c->tol = o.breakdown_tol > 0 ? o.breakdown_tol : (cprec == LOVE_FP64 ? 1e-10 : 1e-6);
        c->k_sample_req = o.k_sample;
        c->n = n_local;
        // a communicator is set up whenever a NCCL id is given (world == 1 runs every
        // collective of the sharded path as an identity; used by the single-GPU tests)
        if (dist && (dist->world > 1 || dist->nccl_unique_id)) {
            if (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world || !dist->nccl_unique_id)
                throw LoveError{LOVE_ERR_ARG, "bad love_dist"};
            c->world = dist->world;
            c->rank = dist->rank;
            nccl_comm_init(*c, dist->nccl_unique_id);
        }
        TempPool tmp(s);
        // global n (k <= n_global); one GPU: the local n, no round trip
        if (c->comm == nullptr) {
            c->n_global = c->n;
        } else {
            int64_t* dn = (int64_t*)tmp.get(sizeof(int64_t));
            cuda_check(cudaMemcpyAsync(dn, &c->n, sizeof(int64_t), cudaMemcpyHostToDevice, s), "n h2d");
            allreduce_sum_i64(*c, dn, 1, s);
            cuda_check(cudaMemcpyAsync(&c->n_global, dn, sizeof(int64_t), cudaMemcpyDeviceToHost, s), "n d2h");
            cuda_check(cudaStreamSynchronize(s), "sync");
        }
        if (c->n_global < 1) throw LoveError{LOVE_ERR_ARG, "no training points"};
        if (k > c->n_global) k = (int32_t)c->n_global;     // a Krylov space has at most n dimensions
        c->k_req = k;
        c->ldq = round_up(std::max<int64_t>(c->n, 1), 4);
    } catch (...) {
        cudaStreamSynchronize(s);
        release(c);
        throw;
    }
    return c;
}

// Lanczos state, the k steps, host copies of T, the cache finish (Rc, mean,
// variance blocks, sampling root).  Leaves the cache complete; throws on numerical errors.
void finish_build(Cache* c, const love_opts& o, int32_t k, cudaStream_t s) {
    const int M = c->g.m_total;
    const size_t vs = c->vsize;
    // ---- Lanczos state
    c->r = dalloc(*c, vs * c->ldq, s);
    c->u = dalloc(*c, sizeof(double) * M, s);
    c->z[0] = dalloc(*c, sizeof(double) * (M + 4), s);      // padded: tiles stage z in 16-byte units
    c->z[1] = dalloc(*c, sizeof(double) * (M + 4), s);
    // column j is streamed at step j (the one-read pass: zero-filled)
    c->Rc_col = c->fused ? dalloc(*c, sizeof(double) * (size_t)M * k, s) : dalloc_unset(*c, sizeof(double) * (size_t)M * k, s);
    c->a = dalloc(*c, sizeof(double) * M, s);
    c->counters = (unsigned long long*)dalloc(*c, sizeof(unsigned long long) * 2, s);
    {
        const size_t K = k;
        const size_t nd = 2 + 3 * (K + 1) + 1 + (K + 1) + 5 * K + 2 + 1;
        c->scal = (double*)dalloc(*c, sizeof(double) * nd, s);
        double* p = c->scal;
        LanczosState& st = c->st;
        st.alpha_cur = p; p += 1;
        st.beta2_cur = p; p += 1;
        st.c_cur = p; p += 3 * (K + 1);     // passes 0, 1 (CGS2) or the one-sync step's three dot vectors
        st.c_len = 3 * (int64_t)(K + 1);
        st.bnorm2 = p; p += 1;
        st.qscale = p; p += K + 1;
        st.alpha = p; p += K;
        st.beta = p; p += K;
        st.Ld = p; p += K;
        st.Ls = p; p += K;
        st.g = p; p += K;
        st.amax_bmax = p; p += 2;
        c->one = p; p += 1;
        st.flags = (int*)dalloc(*c, sizeof(int) * 8, s);
        st.jdev = st.flags + 4;
        st.step_ctr = st.flags + 5;
        if (c->partial) {
            st.omega = (double*)dalloc(*c, sizeof(double) * 3 * (K + 1), s);
            st.pro = (int*)dalloc(*c, sizeof(int) * 4, s);
            const double one = 1.0;                      // omega_{0,0} = q_0^T q_0
            cuda_check(cudaMemcpyAsync(st.omega, &one, sizeof(double), cudaMemcpyHostToDevice, s), "omega init");
            const double eps = c->precision == LOVE_FP64 ? 1.1102230246251565e-16 : 5.9604644775390625e-08;
            st.pro_eps = eps;
            st.pro_tol = o.reorth_tol > 0.0 ? o.reorth_tol : std::sqrt(eps);
        }
        // DGKS-gated second CGS pass (fp64 CGS2, one GPU): the second pass runs only when the
        // first one removed more than 1 - 1/sqrt(2) of the norm (LOVE_NO_DGKS: always)
        if (c->reorth_passes == 2 && c->precision == LOVE_FP64 && c->comm == nullptr && !c->partial && !c->fused &&
            std::getenv("LOVE_NO_DGKS") == nullptr) {
            st.nrm2 = (double*)dalloc(*c, sizeof(double) * 2, s);
            st.dgks = std::getenv("LOVE_DGKS_LATE") ? 1 : 2;   // 2: the first pass decides (dgks_decide)
        }
        if (c->comm == nullptr) {                        // one GPU: spread the dot atomics
            st.crep = 4;                                 // measured: 4 beats 8 and 16 (cfg2, cfg3)
            st.cld = (int)(round_up((int64_t)K + 1, 16) + 16);
            st.c_cur = (double*)dalloc(*c, sizeof(double) * 2 * st.crep * st.cld, s);
            st.c_len = 2 * (int64_t)st.crep * st.cld;
        }
        LOVE_LAUNCH(init_state_kernel, 1, 32, 0, s, st.flags, k, c->one);
    }

    // ---- probe b = (1/m) W_X^T K_UU 1 (average column of K_XU K_UU..., Alg. 1)
    if (c->probe == LOVE_PROBE_AVGCOL) avgcol_probe(*c, s);

    // ---- k Lanczos steps + streamed Cholesky / Rc / mean cache
    if (c->fused) setup_fused(*c, s);
    struct L2Scope {
        void* h;
        ~L2Scope() { l2_persist_end(h); }
    } l2{c->fused ? nullptr : l2_persist_begin(*c, s)};
    host_mark("l2_persist");
    if (c->fused) run_lanczos_fused(*c, s);
    else run_lanczos(*c, s);
    host_mark("lanczos_enqueued");
    // one D2H batch and one synchronisation: flags, |b|^2 and T's alpha_j, beta_j (contiguous
    // in the scalar block) for every j < k
    const size_t K = (size_t)k;
    char* hb = (char*)pinned_scratch(sizeof(int) * 8 + sizeof(double) * (1 + 2 * K) + sizeof(int));
    int* hfl = (int*)hb;
    double* hbn = (double*)(hb + sizeof(int) * 8);
    double* hab = hbn + 1;
    cuda_check(cudaMemcpyAsync(hfl, c->st.flags, sizeof(int) * 8, cudaMemcpyDeviceToHost, s), "flags d2h");
    cuda_check(cudaMemcpyAsync(hbn, c->st.bnorm2, sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaMemcpyAsync(hab, c->st.alpha, sizeof(double) * 2 * K, cudaMemcpyDeviceToHost, s), "T d2h");
    int* hrange = (int*)(hab + 2 * K);
    *hrange = 0;
    if (c->range_flag != nullptr)
        cuda_check(cudaMemcpyAsync(hrange, c->range_flag, sizeof(int), cudaMemcpyDeviceToHost, s), "flag d2h");
    cuda_check(cudaStreamSynchronize(s), "lanczos sync");
    host_mark("lanczos_sync");
    c->range_flag = nullptr;
    if (*hrange) throw LoveError{LOVE_ERR_RANGE, "a training point needs a grid node outside the grid"};
    trace_report(*c, hfl[1]);
    const double bn2 = *hbn;
    cuda_check(cudaGetLastError(), "lanczos kernels");
    if (hfl[3]) throw LoveError{LOVE_ERR_ZERO_PROBE, "the Lanczos probe vector is zero"};
    if (hfl[2]) throw LoveError{LOVE_ERR_NOT_PD, "Cholesky of T_k hit a non-positive pivot"};
    c->k_eff = hfl[1];
    g_launch_count += c->cond_nodes * (hfl[6] / c->cond_steps);   // kernels of the device-terminated step loop
    // LOVE_CACHE_FP64_AUTO (reading A12b): an fp32 Lanczos that broke down before k is not
    // finished -- the caller rebuilds the cache with fp64 factors
    if (o.cache_fp64 == LOVE_CACHE_FP64_AUTO && c->precision == LOVE_FP32 && !c->partial && !c->fused &&
        c->k_eff < c->k_req)
        throw LoveError{kRebuildFp64, "fp32 Lanczos broke down before k: rebuild with an fp64 cache"};
    c->b_norm = std::sqrt(bn2);
    c->n_reorth_steps = std::max(c->k_eff - 1, 0);
    if (c->partial) {
        int pro[4];
        cuda_check(cudaMemcpy(pro, c->st.pro, sizeof(pro), cudaMemcpyDeviceToHost), "pro d2h");
        c->n_reorth_steps = pro[2];
    }
    if (c->st.beta != c->st.alpha + K) throw LoveError{LOVE_ERR_CUDA, "internal: T layout"};
    c->h_alpha.assign(hab, hab + c->k_eff);
    c->h_beta.assign(hab + K, hab + K + std::max(c->k_eff - 1, 0));
    host_mark("alpha_beta");
    if (c->probe == LOVE_PROBE_AVGCOL) mean_cache_eq4(*c, s);   // a = R^T T^{-1} Q^T y
    finish_cache(*c, s);
    c->var_blocks_off = o.var_blocks == LOVE_VAR_BLOCKS_OFF;
    build_var_blocks(*c, s);
    host_mark("finish_enqueued");
    if (c->k_sample_req > 0) build_sampling_cache(*c, s);
    cuda_check(cudaStreamSynchronize(s), "build sync");
    cuda_check(cudaGetLastError(), "build kernels");
}

}  // namespace
}  // namespace love

using namespace love;

extern "C" {

const char* love_last_error(void) { return t_err.c_str(); }
int64_t love_launch_count(void) { return g_launch_count.load(); }
int32_t love_abi_version(void) { return LOVE_ABI_VERSION; }

love_status love_nccl_unique_id(void* out) {
    if (!out) {
        set_error("NULL out");
        return LOVE_ERR_ARG;
    }
    return nccl_get_unique_id(out);
}

static love_status build_grid_once(const love_grid* grid, const love_rbf* rbf, double sigma2, const double* X,
                                   const double* y, int64_t n_local, int32_t k, const love_opts* opts,
                                   const love_dist* dist, void* stream, love_cache** out) {
    Cache* c = nullptr;
    cudaStream_t s = nullptr;
    try {
        if (out) *out = nullptr;
        host_mark("start");
        validate_build(grid, rbf, sigma2, X, y, n_local, k, out);
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        s = work_stream(dev);
        order_after(s, (cudaStream_t)stream);
        const love_opts o = checked_opts(opts);
        c = begin_build(o, sigma2, n_local, k, dist, s);
        GridDev& g = c->g;
        g.d = grid->d;
        g.m_total = 1;
        for (int d = 0; d < 3; ++d) {
            g.m[d] = d < g.d ? (int)grid->m[d] : 1;
            g.lo[d] = d < g.d ? grid->lo[d] : 0.0;
            g.h[d] = d < g.d ? grid->h[d] : 1.0;
        }
        for (int d = g.d - 1, st = 1; d >= 0; --d) {
            g.stride[d] = st;
            st *= g.m[d];
        }
        for (int d = g.d; d < 3; ++d) g.stride[d] = 0;
        for (int d = 0; d < g.d; ++d) g.m_total *= g.m[d];
        c->rbf = *rbf;
        const int M = g.m_total;
        const size_t vs = c->vsize;
        TempPool tmp(s);
        // ---- interpolation records + cell sort
        int* cell = (int*)tmp.get(sizeof(int) * std::max<int64_t>(c->n, 1));
        double* frac64 = (double*)tmp.get(sizeof(double) * std::max<int64_t>(c->n, 1) * g.d);
        int* dflag = (int*)tmp.get(sizeof(int) * 2);
        cuda_check(cudaMemsetAsync(dflag, 0, sizeof(int) * 2, s), "memset");
        c->perm = (int*)dalloc(*c, sizeof(int) * std::max<int64_t>(c->n, 1), s);
        c->cell_start = (int*)dalloc(*c, sizeof(int) * (M + 1), s);
        c->cell_item_start = (int*)dalloc(*c, sizeof(int) * (M + 1), s);
        for (int d = 0; d < g.d; ++d) c->frac[d] = dalloc(*c, vs * (c->ldq + 4), s);   // padded to 16 B units
        if (g.d <= 2 && !c->fused) c->pcell = (int*)dalloc(*c, sizeof(int) * (c->ldq + 4), s);
        // Q~: column j + 1 is written whole (ldq rows) by step j before anything reads it;
        // column 0 (the probe, n rows) is zeroed first so that its padding rows are 0
        // (the one-read pass reads ahead: zero-filled)
        if (c->fused) {
            c->Q = dalloc(*c, vs * c->ldq * (size_t)(k + 1), s);
        } else {
            c->Q = dalloc_unset(*c, vs * c->ldq * (size_t)(k + 1), s);
            cuda_check(cudaMemsetAsync(c->Q, 0, vs * c->ldq, s), "Q0 memset");
        }
        host_mark("begin_build");
        prof_begin(LOVE_PROF_SETUP, s);
        launch_interp_points(*c, X, c->n, cell, frac64, dflag, s);
        if (c->comm != nullptr) {   // the range check is global: every rank must agree before continuing
            float fl = 0.f;
            int hflag = 0;
            cuda_check(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, s), "flag d2h");
            cuda_check(cudaStreamSynchronize(s), "sync");
            {
                float* df = (float*)tmp.get(sizeof(float));
                fl = (float)hflag;
                cuda_check(cudaMemcpyAsync(df, &fl, sizeof(float), cudaMemcpyHostToDevice, s), "h2d");
                allreduce_sum(*c, df, 1, false, s);
                cuda_check(cudaMemcpyAsync(&fl, df, sizeof(float), cudaMemcpyDeviceToHost, s), "d2h");
                cuda_check(cudaStreamSynchronize(s), "sync");
                hflag = fl > 0.f;
            }
            if (hflag) throw LoveError{LOVE_ERR_RANGE, "a training point needs a grid node outside the grid"};
        }
        // probe y: the sorted targets are the first Lanczos column; probe avg: they are kept
        // for the mean cache (Eq. 4) and column 0 is filled below
        if (c->probe == LOVE_PROBE_AVGCOL) c->ysort = dalloc(*c, vs * c->ldq, s);
        launch_counting_sort(*c, cell, frac64, y, c->n, c->probe == LOVE_PROBE_Y ? c->Q : c->ysort, s);
        host_mark("interp+range_sync");
        // the item list (cells cut into <= kItemMax-point chunks) feeds the d >= 2 item kernels and
        // the one-read pass; the d = 1 cell-moment scatter and per-point gather do without it, and
        // then nothing before the Lanczos needs a synchronisation: the range flag is read back
        // with the Lanczos flags (a point off the grid was given cell 0, so every pass stays in
        // bounds until then)
        if (g.d >= 2 || c->fused || c->comm != nullptr) {
            // one GPU: the range flag comes back with the item count (one synchronisation)
            int hrange = 0;
            if (c->comm == nullptr)
                cuda_check(cudaMemcpyAsync(&hrange, dflag, sizeof(int), cudaMemcpyDeviceToHost, s), "flag d2h");
            c->n_items = count_items_host(*c, s);
            if (hrange) throw LoveError{LOVE_ERR_RANGE, "a training point needs a grid node outside the grid"};
            host_mark("sort+items_sync");
            c->item_cell = (int*)dalloc(*c, sizeof(int) * (c->n_items + 8), s);     // padded: staged in 16 B units
            c->item_start = (int*)dalloc(*c, sizeof(int) * (c->n_items + 9), s);
            launch_build_items(*c, s);
            c->M = dalloc(*c, sizeof(double) * (size_t)(1 << (2 * g.d)) * std::max<int64_t>(c->n_items, 1), s);
        } else {
            c->n_items = -1;
            c->range_flag = dflag;
        }
        if (g.d == 1 && !c->fused) c->Mc = dalloc(*c, sizeof(double) * 4 * (size_t)(M + 4), s);
        if (g.d >= 2) {
            c->pullT = dalloc(*c, sizeof(double) * (size_t)(g.d == 2 ? 4 : 16) * M, s);
            if (g.d == 3) c->pullV = dalloc(*c, sizeof(double) * 4 * (size_t)M, s);
        }

        // ---- K_UU
        setup_kuu(*c, s);
        prof_end(LOVE_PROF_SETUP, s);

        host_mark("setup_kuu");
        finish_build(c, o, k, s);
        host_mark("finish");
        host_marks_flush();
        *out = reinterpret_cast<love_cache*>(c);
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        if (c) {
            if (s) cudaStreamSynchronize(s);
            release(c);
        }
        return fail(e);
    }
}

static love_status build_additive_once(const love_axis* axes, int32_t d, double sigma2, const double* X,
                                       const double* y, int64_t n_local, int32_t k, const love_opts* opts,
                                       const love_dist* dist, void* stream, love_cache** out) {
    Cache* c = nullptr;
    cudaStream_t s = nullptr;
    try {
        if (out) *out = nullptr;
        if (!axes || !out) throw LoveError{LOVE_ERR_ARG, "NULL axes/out"};
        if (d < 1 || d > LOVE_MAX_ADDITIVE) throw LoveError{LOVE_ERR_ARG, "d must be 1..LOVE_MAX_ADDITIVE"};
        int64_t mt = 0;
        for (int e = 0; e < d; ++e) {
            const love_axis& x = axes[e];
            if (x.m < 4 || x.m > 1024) throw LoveError{LOVE_ERR_ARG, "axis m must be 4..1024"};
            if (!(x.h > 0.0) || !std::isfinite(x.lo) || !(x.lengthscale > 0.0) || !(x.outputscale > 0.0))
                throw LoveError{LOVE_ERR_ARG, "axis h, lengthscale, outputscale must be > 0 and lo finite"};
            mt += x.m;
        }
        if (!(sigma2 > 0.0)) throw LoveError{LOVE_ERR_ARG, "sigma^2 must be > 0"};
        if (k < 1 || k > 2048) throw LoveError{LOVE_ERR_ARG, "k must be 1..2048"};
        if (n_local < 0 || n_local >= (int64_t(1) << 31)) throw LoveError{LOVE_ERR_ARG, "bad n_local"};
        if (n_local > 0 && (!X || !y)) throw LoveError{LOVE_ERR_ARG, "NULL X/y"};
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        s = work_stream(dev);
        order_after(s, (cudaStream_t)stream);
        love_opts o = checked_opts(opts);
        if (o.k_sample > 0) throw LoveError{LOVE_ERR_ARG, "k_sample is not supported for additive caches"};
        if (o.lanczos_mode == LOVE_LANCZOS_ONE_READ)
            throw LoveError{LOVE_ERR_ARG, "the one-read Lanczos pass is grid-only"};
        if (o.lanczos_mode != LOVE_LANCZOS_PARTIAL) o.lanczos_mode = LOVE_LANCZOS_TWO_PASS;
        c = begin_build(o, sigma2, n_local, k, dist, s);
        c->fused = false;
        c->additive = true;
        AddDev& a = c->ad;
        a.d = d;
        a.off[0] = 0;
        for (int e = 0; e < d; ++e) {
            a.m[e] = (int)axes[e].m;
            a.lo[e] = axes[e].lo;
            a.h[e] = axes[e].h;
            a.ls[e] = axes[e].lengthscale;
            a.s2[e] = axes[e].outputscale;
            a.off[e + 1] = a.off[e] + a.m[e];
            for (int i = 0; i < 4; ++i) {
                const double r = (double)i * a.h[e];
                a.c4[e][i] = std::exp(-(r * r) / (2.0 * a.ls[e] * a.ls[e]));
            }
        }
        c->g = GridDev{};
        c->g.d = 0;
        c->g.m_total = (int)mt;
        c->rbf = love_rbf{};
        c->rbf.outputscale = 1.0;
        const size_t vs = c->vsize;
        TempPool tmp(s);
        int* dflag = (int*)tmp.get(sizeof(int) * 2);
        cuda_check(cudaMemsetAsync(dflag, 0, sizeof(int) * 2, s), "memset");
        // Q~: column j + 1 is written whole (ldq rows) by step j before anything reads it;
        // column 0 (the probe, n rows) is zeroed first so that its padding rows are 0
        // (the one-read pass reads ahead: zero-filled)
        if (c->fused) {
            c->Q = dalloc(*c, vs * c->ldq * (size_t)(k + 1), s);
        } else {
            c->Q = dalloc_unset(*c, vs * c->ldq * (size_t)(k + 1), s);
            cuda_check(cudaMemsetAsync(c->Q, 0, vs * c->ldq, s), "Q0 memset");
        }
        prof_begin(LOVE_PROF_SETUP, s);
        additive_setup(*c, X, y, dflag, s);
        {   // the range check is global: every rank must agree before continuing
            int hflag = 0;
            cuda_check(cudaMemcpyAsync(&hflag, dflag, sizeof(int), cudaMemcpyDeviceToHost, s), "flag d2h");
            cuda_check(cudaStreamSynchronize(s), "sync");
            if (c->comm != nullptr) {
                float fl = (float)hflag;
                float* df = (float*)tmp.get(sizeof(float));
                cuda_check(cudaMemcpyAsync(df, &fl, sizeof(float), cudaMemcpyHostToDevice, s), "h2d");
                allreduce_sum(*c, df, 1, false, s);
                cuda_check(cudaMemcpyAsync(&fl, df, sizeof(float), cudaMemcpyDeviceToHost, s), "d2h");
                cuda_check(cudaStreamSynchronize(s), "sync");
                hflag = fl > 0.f;
            }
            if (hflag) throw LoveError{LOVE_ERR_RANGE, "a training point needs a grid node outside its component grid"};
        }
        // probe y: the targets (original order) are the first Lanczos column; probe avg: kept
        // for the mean cache (Eq. 4) and column 0 is filled by the probe
        void* ydst = c->Q;
        if (c->probe == LOVE_PROBE_AVGCOL) ydst = c->ysort = dalloc(*c, vs * c->ldq, s);
        if (c->n > 0) {
            if (c->precision == LOVE_FP64)
                cuda_check(cudaMemcpyAsync(ydst, y, sizeof(double) * c->n, cudaMemcpyDeviceToDevice, s), "y copy");
            else
                launch_convert<double, float>(y, (float*)ydst, c->n, s);
        }
        c->n_items = c->n;
        prof_end(LOVE_PROF_SETUP, s);
        finish_build(c, o, k, s);
        *out = reinterpret_cast<love_cache*>(c);
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        if (c) {
            if (s) cudaStreamSynchronize(s);
            release(c);
        }
        return fail(e);
    }
}

// LOVE_CACHE_FP64_AUTO (reading A12b): an fp32 Lanczos that breaks down before k has reached
// the point where its fp32 vectors no longer resolve beta_j (tau = 1e-6 ~ 16 eps_32 of ||T||):
// the problem is converged (var << prior) and the late fp32 directions are round-off.  The fp32
// build stops right after its Lanczos loop (finish_build throws kRebuildFp64) and the cache is
// rebuilt with fp64 factors (the outputs stay fp32), which runs to the fp64 breakdown the
// oracle sees.  Every rank sees the same k_eff, so they all take the same branch.

static love_opts with_fp64_cache(const love_opts* opts) {
    love_opts o{};
    if (opts) o = *opts;
    o.cache_fp64 = LOVE_CACHE_FP64_ON;
    return o;
}

love_status love_build_cache(const love_grid* grid, const love_rbf* rbf, double sigma2, const double* X,
                             const double* y, int64_t n_local, int32_t k, const love_opts* opts,
                             const love_dist* dist, void* stream, love_cache** out) {
    love_status st = build_grid_once(grid, rbf, sigma2, X, y, n_local, k, opts, dist, stream, out);
    if (st == kRebuildFp64) {
        const love_opts o = with_fp64_cache(opts);
        st = build_grid_once(grid, rbf, sigma2, X, y, n_local, k, &o, dist, stream, out);
    }
    return st;
}

love_status love_build_cache_additive(const love_axis* axes, int32_t d, double sigma2, const double* X,
                                      const double* y, int64_t n_local, int32_t k, const love_opts* opts,
                                      const love_dist* dist, void* stream, love_cache** out) {
    love_status st = build_additive_once(axes, d, sigma2, X, y, n_local, k, opts, dist, stream, out);
    if (st == kRebuildFp64) {
        const love_opts o = with_fp64_cache(opts);
        st = build_additive_once(axes, d, sigma2, X, y, n_local, k, &o, dist, stream, out);
    }
    return st;
}

void love_free(love_cache* cache) { release(reinterpret_cast<Cache*>(cache)); }

love_status love_cache_info(const love_cache* cache, love_info* info) {
    try {
        if (!cache || !info) throw LoveError{LOVE_ERR_ARG, "NULL cache/info"};
        const Cache* c = reinterpret_cast<const Cache*>(cache);
        cuda_check(cudaDeviceSynchronize(), "sync");
        unsigned long long cnt[2];
        cuda_check(cudaMemcpy(cnt, c->counters, sizeof(cnt), cudaMemcpyDeviceToHost), "counters d2h");
        std::memset(info, 0, sizeof(*info));
        info->k_eff = c->k_eff;
        info->n_reorth_steps = c->n_reorth_steps;
        info->k_pad = c->k_pad;
        info->k_sample_eff = c->k_sample_eff;
        info->precision = c->out_precision;
        info->cache_precision = c->precision;
        info->n_local = c->n;
        info->n_global = c->n_global;
        info->m_total = c->g.m_total;
        info->n_items = c->n_items;
        if (c->n_items < 0) {   // not listed at build time: the count of the per-cell item scan
            int nit = 0;
            cuda_check(cudaMemcpy(&nit, c->cell_item_start + c->g.m_total, sizeof(int), cudaMemcpyDeviceToHost),
                       "items d2h");
            info->n_items = nit;
        }
        info->b_norm = c->b_norm;
        info->alpha = c->h_alpha.data();
        info->beta = c->h_beta.data();
        info->n_negative_var = (int64_t)cnt[0];
        info->n_out_of_range = (int64_t)cnt[1];
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        return fail(e);
    }
}

love_status love_predict_var(const love_cache* cache, const double* Xs, int64_t t, void* var_out, void* mean_out,
                             void* stream) {
    try {
        if (!cache || (t > 0 && (!Xs || !var_out)) || t < 0) throw LoveError{LOVE_ERR_ARG, "bad arguments"};
        const Cache* c = reinterpret_cast<const Cache*>(cache);
        cudaStream_t s = (cudaStream_t)stream;
        if (c->precision == LOVE_FP64 && c->out_precision == LOVE_FP32) {
            // fp64 cache, fp32 outputs (opts.cache_fp64): fp64 results rounded once
            TempPool tmp(s);
            double* v64 = (double*)tmp.get(sizeof(double) * t);
            double* m64 = mean_out ? (double*)tmp.get(sizeof(double) * t) : nullptr;
            launch_predict<double>(*c, Xs, nullptr, t, v64, m64, s);
            launch_convert<double, float>(v64, (float*)var_out, t, s);
            if (mean_out) launch_convert<double, float>(m64, (float*)mean_out, t, s);
        } else if (c->precision == LOVE_FP64) {
            launch_predict<double>(*c, Xs, nullptr, t, (double*)var_out, (double*)mean_out, s);
        } else {
            launch_predict<float>(*c, Xs, nullptr, t, (float*)var_out, (float*)mean_out, s);
        }
        cuda_check(cudaGetLastError(), "predict_var launch");
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        return fail(e);
    }
}

love_status love_predict_covar(const love_cache* cache, const double* Xa, const double* Xb, int64_t t,
                               void* cov_out, void* stream) {
    try {
        if (!cache || (t > 0 && (!Xa || !Xb || !cov_out)) || t < 0) throw LoveError{LOVE_ERR_ARG, "bad arguments"};
        const Cache* c = reinterpret_cast<const Cache*>(cache);
        cudaStream_t s = (cudaStream_t)stream;
        if (c->precision == LOVE_FP64 && c->out_precision == LOVE_FP64) {
            launch_predict<double>(*c, Xa, Xb, t, (double*)cov_out, nullptr, s);
        } else if (t > 0) {
            // fp32 outputs: the pair products (Rc^T w_a) . (Rc^T w_b) ~ prior cancel against the
            // prior, so they are formed from fp64 rows (an fp64 cache, or the fp64 row copy of
            // an fp32 cache's Rc) and the fp64 covariance is rounded once
            Cache w = *c;
            w.allocs.clear();
            if (c->precision == LOVE_FP32) {
                w.Rc = rc_rows64(*c, s);
                w.precision = LOVE_FP64;
                w.vsize = 8;
            }
            TempPool tmp(s);
            double* c64 = (double*)tmp.get(sizeof(double) * t);
            launch_predict<double>(w, Xa, Xb, t, c64, nullptr, s);
            launch_convert<double, float>(c64, (float*)cov_out, t, s);
        }
        cuda_check(cudaGetLastError(), "predict_covar launch");
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        return fail(e);
    }
}

love_status love_sample(const love_cache* cache, const double* Xs, int64_t t, int64_t ns, uint64_t seed,
                        const double* zeta, void* out, void* stream) {
    try {
        if (!cache || t < 0 || ns < 0 || ((t > 0 && ns > 0) && (!Xs || !out)))
            throw LoveError{LOVE_ERR_ARG, "bad arguments"};
        const Cache* c = reinterpret_cast<const Cache*>(cache);
        if (c->k_sample_eff <= 0 || c->S == nullptr)
            throw LoveError{LOVE_ERR_STATE, "cache was built without a sampling root (k_sample = 0)"};
        cudaStream_t s = (cudaStream_t)stream;
        if (c->out_precision == LOVE_FP64) launch_sample<double>(*c, Xs, t, ns, seed, zeta, (double*)out, s);
        else launch_sample<float>(*c, Xs, t, ns, seed, zeta, (float*)out, s);
        cuda_check(cudaGetLastError(), "sample launch");
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        return fail(e);
    }
}

love_status love_ski_mvm(const love_cache* cache, const void* v, void* out, void* stream) {
    try {
        if (!cache || !v || !out) throw LoveError{LOVE_ERR_ARG, "NULL argument"};
        const Cache* c = reinterpret_cast<const Cache*>(cache);
        if (c->world > 1) throw LoveError{LOVE_ERR_STATE, "love_ski_mvm needs a single-rank cache"};
        cudaStream_t s = (cudaStream_t)stream;
        TempPool tmp(s);
        Cache w = *c;   // shallow copy with private scratch
        w.allocs.clear();
        const size_t vs = c->vsize;
        void* vsrt = tmp.get(vs * c->ldq);
        void* rs = tmp.get(vs * c->ldq);
        double* u = (double*)tmp.get(sizeof(double) * c->g.m_total);
        double* z = (double*)tmp.get(sizeof(double) * c->g.m_total);
        w.M = tmp.get(sizeof(double) * (size_t)(1 << (2 * c->g.d)) * std::max<int64_t>(c->n_items, 1));
        if (c->fft_buf) w.fft_buf = tmp.get(sizeof(double2) * c->fft_N);
        if (c->ktmp[0]) {
            w.ktmp[0] = tmp.get(sizeof(double) * c->g.m_total);
            w.ktmp[1] = tmp.get(sizeof(double) * c->g.m_total);
        }
        if (c->precision == LOVE_FP64) {
            launch_permute<double>(w, (const double*)v, (double*)vsrt, true, s);
            const StepRef ref{nullptr, 0, c->one, nullptr};
            launch_scatter<double>(w, (const double*)vsrt, ref, u, s);
            launch_kuu(w, u, z, s);
            launch_gather<double>(w, z, (const double*)vsrt, ref, (double*)rs, nullptr, s);
            launch_permute<double>(w, (const double*)rs, (double*)out, false, s);
        } else {
            launch_permute<float>(w, (const float*)v, (float*)vsrt, true, s);
            const StepRef ref{nullptr, 0, c->one, nullptr};
            launch_scatter<float>(w, (const float*)vsrt, ref, u, s);
            launch_kuu(w, u, z, s);
            launch_gather<float>(w, z, (const float*)vsrt, ref, (float*)rs, nullptr, s);
            launch_permute<float>(w, (const float*)rs, (float*)out, false, s);
        }
        cuda_check(cudaGetLastError(), "ski_mvm launch");
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        return fail(e);
    }
}

love_status love_kuu_mvm(const love_cache* cache, const void* u, void* out, void* stream) {
    try {
        if (!cache || !u || !out) throw LoveError{LOVE_ERR_ARG, "NULL argument"};
        const Cache* c = reinterpret_cast<const Cache*>(cache);
        cudaStream_t s = (cudaStream_t)stream;
        TempPool tmp(s);
        Cache w = *c;
        w.allocs.clear();
        if (c->fft_buf) w.fft_buf = tmp.get(sizeof(double2) * c->fft_N);
        if (c->ktmp[0]) {
            w.ktmp[0] = tmp.get(sizeof(double) * c->g.m_total);
            w.ktmp[1] = tmp.get(sizeof(double) * c->g.m_total);
        }
        if (c->precision == LOVE_FP64) {
            launch_kuu(w, (const double*)u, (double*)out, s);
        } else {
            double* ud = (double*)tmp.get(sizeof(double) * c->g.m_total);
            double* zd = (double*)tmp.get(sizeof(double) * c->g.m_total);
            launch_convert<float, double>((const float*)u, ud, c->g.m_total, s);
            launch_kuu(w, ud, zd, s);
            launch_convert<double, float>(zd, (float*)out, c->g.m_total, s);
        }
        cuda_check(cudaGetLastError(), "kuu_mvm launch");
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        return fail(e);
    }
}

love_status love_cache_export(const love_cache* cache, int32_t what, void* dst, int64_t capacity, int64_t* bytes,
                              void* stream) {
    try {
        if (!cache) throw LoveError{LOVE_ERR_ARG, "NULL cache"};
        const Cache* c = reinterpret_cast<const Cache*>(cache);
        const void* src = nullptr;
        int64_t nb = 0;
        switch (what) {
            case LOVE_EXPORT_RC: src = c->Rc; nb = (int64_t)c->vsize * c->g.m_total * c->k_pad; break;
            case LOVE_EXPORT_MEAN: src = c->a; nb = (int64_t)sizeof(double) * c->g.m_total; break;
            case LOVE_EXPORT_S: src = c->S; nb = (int64_t)c->vsize * c->g.m_total * c->ks_pad; break;
            case LOVE_EXPORT_PERM: src = c->perm; nb = (int64_t)sizeof(int) * c->n; break;
            default: throw LoveError{LOVE_ERR_ARG, "unknown export"};
        }
        if (bytes) *bytes = nb;
        if (!dst) return LOVE_OK;
        if (capacity < nb) throw LoveError{LOVE_ERR_ARG, "destination too small"};
        if (!src || nb == 0) return LOVE_OK;
        cuda_check(cudaMemcpyAsync(dst, src, nb, cudaMemcpyDeviceToDevice, (cudaStream_t)stream), "export copy");
        return LOVE_OK;
    } catch (...) {
        const LoveError e = current_error();
        return fail(e);
    }
}

}  // extern "C"
