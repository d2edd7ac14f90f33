// common.cuh -- shared device helpers of the LOVE sm_100a library (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <utility>
#include <string>

namespace love {

extern std::atomic<int64_t> g_launch_count;

// Programmatic dependent launch (PDL).  Inside a PdlScope every LOVE_LAUNCH carries the
// programmatic-stream-serialization attribute: the next kernel's CTAs may be scheduled while
// the previous grid drains, and they block in pdl_wait() (griddepcontrol.wait: the previous
// grid has completed and its writes are visible) before touching anything it produced.
// Every kernel launched inside a PdlScope must therefore call pdl_wait() first.
extern thread_local bool t_pdl;
struct PdlScope {
    bool prev;
    explicit PdlScope(bool on) : prev(t_pdl) { t_pdl = on; }
    ~PdlScope() { t_pdl = prev; }
};
// Inside a DoneScope the K_UU kernels get the Lanczos `done` flag and return at once when it
// is set: steps launched past a breakdown (graph replays are fixed) then cost only launches.
extern thread_local const int* t_done;
struct DoneScope {
    const int* prev;
    explicit DoneScope(const int* f) : prev(t_done) { t_done = f; }
    ~DoneScope() { t_done = prev; }
};
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// ---- in-pipeline kernel trace (liblove_trace.so with LOVE_TRACE=1): per (step j, kernel id) the
// earliest CTA start after griddepcontrol.wait, from %globaltimer (ns), recorded by thread 0 of
// every CTA (a kernel's slot = the next kernel's start - its start; start only, so that the
// streaming kernels keep their register allocation).  Each translation unit holds its own device pointer
// (LOVE_TRACE_TU), bound stream-ordered around the Lanczos replays; nullptr = off (one load
// and a branch per CTA).
constexpr int kTraceKernels = 16;
enum TraceKid {
    kTrMoments = 0, kTrPullLast = 1, kTrPullMid = 2, kTrPullFirst = 3, kTrFft0 = 4, kTrFft1 = 5, kTrFft2 = 6,
    kTrGather = 7, kTrDots0 = 8, kTrUpdate0 = 9, kTrDots1 = 10, kTrUpdate1 = 11, kTrNodepass = 12,
    kTrArrive = 13, kTrAdvanced = 14,  // update's CTAs at the step counter [first, last]; the last CTA done
    kTrSampV = 15                      // sampling Lanczos: v = z - Rc t (its step head is kTrMoments)
};
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_start(unsigned long long* base, int kid, int j) {
    if (base != nullptr && threadIdx.x == 0 && threadIdx.y == 0)
        atomicMin(base + ((size_t)j * kTraceKernels + kid) * 2, gtimer());
}
__device__ __forceinline__ void trace_arrive(unsigned long long* base, int kid, int j) {
    if (base != nullptr && threadIdx.x == 0 && threadIdx.y == 0) {
        const unsigned long long t = gtimer();
        atomicMin(base + ((size_t)j * kTraceKernels + kid) * 2, t);
        atomicMax(base + ((size_t)j * kTraceKernels + kid) * 2 + 1, t);
    }
}
#define LOVE_TRACE_TU(name)                                                                   \
    static __device__ unsigned long long* g_love_trace = nullptr;                            \
    void trace_bind_##name(unsigned long long* p, cudaStream_t s) {                          \
        cudaMemcpyToSymbolAsync(g_love_trace, &p, sizeof(p), 0, cudaMemcpyHostToDevice, s); \
    }
// compiled in only for the measurement build (make trace -> liblove_trace.so, -DLOVE_TRACE_ON)
#ifdef LOVE_TRACE_ON
#define LOVE_TRACE(kid, j) ::love::trace_start(g_love_trace, (kid), (j))
#define LOVE_TRACE_ARRIVE(kid, j) ::love::trace_arrive(g_love_trace, (kid), (j))
#else
#define LOVE_TRACE(kid, j) \
    do {                   \
    } while (0)
#define LOVE_TRACE_ARRIVE(kid, j) \
    do {                          \
    } while (0)
#endif
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                      Args&&... args) {
    if (!t_pdl) {
        kernel<<<grid, block, smem, stream>>>(std::forward<Args>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#define LOVE_LAUNCH(kernel, grid, block, smem, stream, ...)                         \
    do {                                                                            \
        ::love::launch_ex(kernel, dim3(grid), dim3(block), (size_t)(smem), (stream), __VA_ARGS__); \
        ::love::g_launch_count.fetch_add(1, std::memory_order_relaxed);              \
    } while (0)

constexpr int kWarp = 32;
constexpr int kItemMax = 32;  // max points per interpolation work item (one cell chunk)

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// Keys cubic-convolution weights, a = -1/2 (reading A2): for a point at u_j + f*h
// the nodes j-1, j, j+1, j+2 get u(1+f), u(f), u(1-f), u(2-f).  Written as the cubic
// polynomials in f that these evaluate to (same values, fewer operations):
//   u(1+f) = -0.5 f^3 +     f^2 - 0.5 f
//   u(f)   =  1.5 f^3 - 2.5 f^2         + 1
//   u(1-f) = -1.5 f^3 + 2   f^2 + 0.5 f
//   u(2-f) =  0.5 f^3 - 0.5 f^2
template <typename T>
__device__ __forceinline__ void keys4(T f, T w[4]) {
    const T f2 = f * f, f3 = f2 * f;
    w[0] = T(-0.5) * f3 + f2 - T(0.5) * f;
    w[1] = T(1.5) * f3 - T(2.5) * f2 + T(1);
    w[2] = T(-1.5) * f3 + T(2) * f2 + T(0.5) * f;
    w[3] = T(0.5) * f3 - T(0.5) * f2;
}

// single Keys weight: slot 0..3 of keys4 (nodes j-1, j, j+1, j+2), branch-free
template <typename T>
__device__ __forceinline__ T keys1(T f, int slot) {
    // coefficients (f^3, f^2, f^1, f^0) of the four cubics of keys4, packed per slot
    const T c3 = slot == 0 ? T(-0.5) : slot == 1 ? T(1.5) : slot == 2 ? T(-1.5) : T(0.5);
    const T c2 = slot == 0 ? T(1) : slot == 1 ? T(-2.5) : slot == 2 ? T(2) : T(-0.5);
    const T c1 = slot == 0 ? T(-0.5) : slot == 2 ? T(0.5) : T(0);
    const T c0 = slot == 1 ? T(1) : T(0);
    return ((c3 * f + c2) * f + c1) * f + c0;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum (blockDim.x multiple of 32, <= 1024); result valid in thread 0.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* smem32) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) smem32[wid] = v;
    __syncthreads();
    T r = T(0);
    if (wid == 0) {
        r = (lane < (int)(blockDim.x >> 5)) ? smem32[lane] : T(0);
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

template <typename V> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };

}  // namespace love
