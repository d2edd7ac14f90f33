// profile.cpp -- phase timing with CUDA events on the launching stream (love_profile_*), and
// NVTX ranges over the same phases for external profilers (LOVE_NVTX=1: ncu --nvtx
// --nvtx-include "love.reorth_update/" ..., header-only NVTX v3, no library to link).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "love_internal.h"

namespace love {

namespace {
struct Pending {
    int cat;
    cudaEvent_t a, b;
};
struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<Pending> pending;
    double ms[LOVE_PROF_N] = {0};
    int64_t calls[LOVE_PROF_N] = {0};
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};
Profiler& prof() {
    static Profiler p;
    return p;
}
thread_local cudaEvent_t t_open[LOVE_PROF_N] = {nullptr};
}  // namespace

bool profiling() { return prof().on; }

// ---- in-pipeline kernel trace (LOVE_TRACE=1, common.cuh)
void trace_begin(Cache& c, int k, cudaStream_t s) {
#ifdef LOVE_TRACE_ON
    static const bool on = std::getenv("LOVE_TRACE") != nullptr;
#else
    const bool on = false;
#endif
    if (!on || k < 1) return;
    const size_t rows = (size_t)k * kTraceKernels;
    c.trace = (unsigned long long*)dalloc_unset(c, rows * 2 * sizeof(unsigned long long), s);
    cuda_check(cudaMemsetAsync(c.trace, 0, rows * 2 * sizeof(unsigned long long), s), "trace memset");
    cuda_check(cudaMemset2DAsync(c.trace, 2 * sizeof(unsigned long long), 0xff, sizeof(unsigned long long), rows, s),
               "trace memset");
    trace_bind_ski(c.trace, s);
    trace_bind_kuu(c.trace, s);
    trace_bind_lanczos(c.trace, s);
    trace_bind_sample(c.trace, s);
}

void trace_end(cudaStream_t s) {
    trace_bind_ski(nullptr, s);
    trace_bind_kuu(nullptr, s);
    trace_bind_lanczos(nullptr, s);
    trace_bind_sample(nullptr, s);
}

// One JSON line on stderr: per kernel id its mean slot (its first CTA start after the wait to
// the next kernel's first start, the next step's first kernel for the last one), over the steps
// 2 .. k_eff - 3, and the mean step period.
void trace_report(Cache& c, int k_eff) {
    if (c.trace == nullptr) return;
    static const char* names[kTraceKernels] = {"moments", "pull_last", "pull_mid", "pull_first", "fft0", "fft1",
                                               "fft2", "gather", "dots0", "update0", "dots1", "update1",
                                               "nodepass", "k13", "k14", "samp_v"};
    const int k = k_eff;
    std::vector<unsigned long long> h((size_t)k * kTraceKernels * 2);
    cuda_check(cudaMemcpy(h.data(), c.trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost),
               "trace d2h");
    const unsigned long long kNone = ~0ull;
    auto starts = [&](int j) {
        std::vector<std::pair<unsigned long long, int>> o;
        const unsigned long long* r = h.data() + (size_t)j * kTraceKernels * 2;
        for (int q = 0; q < kTraceKernels; ++q)
            if (r[2 * q] != kNone && q != kTrArrive && q != kTrAdvanced) o.push_back({r[2 * q], q});
        std::sort(o.begin(), o.end());
        return o;
    };
    double slot[kTraceKernels] = {0};
    int cnt[kTraceKernels] = {0};
    double period = 0.0;
    int np = 0;
    // the step's advancing update: its start -> first CTA at the counter -> last CTA at the
    // counter -> the last CTA's scalars done -> the next step's first kernel start
    double adv[4] = {0, 0, 0, 0};
    int na = 0;
    for (int j = 2; j + 3 < k; ++j) {
        const auto o = starts(j), on = starts(j + 1);
        if (o.empty() || on.empty()) continue;
        const unsigned long long* r = h.data() + (size_t)j * kTraceKernels * 2;
        if (r[2 * kTrArrive] != kNone && r[2 * kTrAdvanced] != kNone) {
            const unsigned long long us = o.back().first;      // the last kernel of the step
            adv[0] += (double)((long long)r[2 * kTrArrive] - (long long)us);
            adv[1] += (double)(r[2 * kTrArrive + 1] - r[2 * kTrArrive]);
            adv[2] += (double)((long long)r[2 * kTrAdvanced] - (long long)r[2 * kTrArrive + 1]);
            adv[3] += (double)((long long)on[0].first - (long long)r[2 * kTrAdvanced]);
            ++na;
        }
        for (size_t i = 0; i < o.size(); ++i) {
            const unsigned long long nxt = i + 1 < o.size() ? o[i + 1].first : on[0].first;
            slot[o[i].second] += (double)(nxt - o[i].first);
            cnt[o[i].second] += 1;
        }
        period += (double)(on[0].first - o[0].first);
        ++np;
    }
    std::string out = "{\"trace\": {\"steps\": " + std::to_string(np) + ", \"period_us\": " +
                      std::to_string(np ? period / np / 1000.0 : 0.0) + ", \"slot_us\": {";
    bool first = true;
    for (int q = 0; q < kTraceKernels; ++q) {
        if (!cnt[q]) continue;
        out += std::string(first ? "" : ", ") + "\"" + names[q] + "\": " + std::to_string(slot[q] / cnt[q] / 1000.0);
        first = false;
    }
    out += "}";
    if (na)
        out += ", \"advance_us\": {\"to_first_arrival\": " + std::to_string(adv[0] / na / 1000.0) +
               ", \"arrival_spread\": " + std::to_string(adv[1] / na / 1000.0) + ", \"last_cta_scalars\": " +
               std::to_string(adv[2] / na / 1000.0) + ", \"to_next_kernel\": " + std::to_string(adv[3] / na / 1000.0) +
               "}";
    out += "}}";
    std::fprintf(stderr, "%s\n", out.c_str());
    c.trace = nullptr;                           // the buffer stays with the cache's allocations
}


namespace {
struct HostMarks {
    bool on = std::getenv("LOVE_HOST_TIMING") != nullptr;
    std::vector<std::pair<const char*, std::chrono::steady_clock::time_point>> m;
};
HostMarks& marks() {
    thread_local HostMarks h;
    return h;
}
}  // namespace

cudaGraphExec_t graph_exec_cached(cudaGraph_t g, const std::string& key) {
    thread_local std::unordered_map<std::string, cudaGraphExec_t> cache;
    static const bool off = std::getenv("LOVE_NO_GRAPH_CACHE") != nullptr;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    const std::string k = key + "/dev" + std::to_string(dev);
    if (!off) {
        auto it = cache.find(k);
        if (it != cache.end()) {
            cudaGraphExecUpdateResultInfo info;
            if (cudaGraphExecUpdate(it->second, g, &info) == cudaSuccess) return it->second;
            (void)cudaGetLastError();
            cudaGraphExecDestroy(it->second);
            cache.erase(it);
        }
    }
    cudaGraphExec_t ge = nullptr;
    cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
    if (!off) cache[k] = ge;
    return ge;
}

void host_mark(const char* what) {
    HostMarks& h = marks();
    if (h.on) h.m.emplace_back(what, std::chrono::steady_clock::now());
}

void host_marks_flush() {
    HostMarks& h = marks();
    if (!h.on || h.m.empty()) return;
    std::fprintf(stderr, "[love host]");
    for (size_t i = 1; i < h.m.size(); ++i)
        std::fprintf(stderr, " %s %.1f", h.m[i].first,
                     std::chrono::duration<double, std::micro>(h.m[i].second - h.m[i - 1].second).count());
    std::fprintf(stderr, " | total %.1f us\n",
                 std::chrono::duration<double, std::micro>(h.m.back().second - h.m.front().second).count());
    h.m.clear();
}

namespace {
const char* const kNvtxNames[LOVE_PROF_N] = {"love.setup", "love.scatter", "love.kuu", "love.gather",
                                             "love.reorth_dots", "love.reorth_update", "love.scalars_rc",
                                             "love.finish", "love.query", "love.sample_cache", "love.sample",
                                             "love.comm", "love.fused_pass", "love.sample_gemm"};
bool nvtx_on() {
    static const bool v = std::getenv("LOVE_NVTX") != nullptr && std::atoi(std::getenv("LOVE_NVTX")) != 0;
    return v;
}
}  // namespace

void prof_begin(int cat, cudaStream_t s) {
    if (nvtx_on() && cat >= 0 && cat < LOVE_PROF_N) nvtxRangePushA(kNvtxNames[cat]);
    Profiler& p = prof();
    if (!p.on) return;
    std::lock_guard<std::mutex> g(p.mu);
    cudaEvent_t e = p.get();
    cudaEventRecord(e, s);
    t_open[cat] = e;
}

void prof_end(int cat, cudaStream_t s) {
    if (nvtx_on() && cat >= 0 && cat < LOVE_PROF_N) nvtxRangePop();
    Profiler& p = prof();
    if (!p.on || t_open[cat] == nullptr) return;
    std::lock_guard<std::mutex> g(p.mu);
    cudaEvent_t e = p.get();
    cudaEventRecord(e, s);
    p.pending.push_back({cat, t_open[cat], e});
    t_open[cat] = nullptr;
}

}  // namespace love

using namespace love;

extern "C" {

void love_profile_enable(int32_t on) { prof().on = on != 0; }

love_status love_profile_read(double* ms_out, int64_t* calls_out, int32_t reset) {
    Profiler& p = prof();
    std::lock_guard<std::mutex> g(p.mu);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        set_error("cudaDeviceSynchronize failed in love_profile_read");
        return LOVE_ERR_CUDA;
    }
    for (const Pending& q : p.pending) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, q.a, q.b) == cudaSuccess) {
            p.ms[q.cat] += t;
            p.calls[q.cat] += 1;
        }
        p.pool.push_back(q.a);
        p.pool.push_back(q.b);
    }
    p.pending.clear();
    for (int i = 0; i < LOVE_PROF_N; ++i) {
        if (ms_out) ms_out[i] = p.ms[i];
        if (calls_out) calls_out[i] = p.calls[i];
        if (reset) {
            p.ms[i] = 0;
            p.calls[i] = 0;
        }
    }
    return LOVE_OK;
}

}  // extern "C"
