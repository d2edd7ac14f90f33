// profile.cpp -- phase timing with CUDA events on the launching stream (love_profile_*).
#include <cuda_runtime.h>

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

void prof_begin(int cat, cudaStream_t s) {
    Profiler& p = prof();
    if (!p.on) return;
    std::lock_guard<std::mutex> g(p.mu);
    cudaEvent_t e = p.get();
    cudaEventRecord(e, s);
    t_open[cat] = e;
}

void prof_end(int cat, cudaStream_t s) {
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
