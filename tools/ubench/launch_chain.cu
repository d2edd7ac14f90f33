// Per-kernel cost of a dependent chain on B200: CUDA graph of K small kernels (plain, PDL
// wait, PDL wait+trigger) vs one persistent kernel with K grid barriers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_chain tools/ubench/launch_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void wait_() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void trig_() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// each thread touches a few bytes of a buffer so the kernel is not empty
template <int MODE>
__global__ void step_kernel(float* buf, int n) {
    if (MODE >= 1) wait_();
    if (MODE == 2) trig_();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) buf[i] += 1.0f;
}

__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;

__global__ void persistent_kernel(float* buf, int n, int K) {
    for (int it = 0; it < K; ++it) {
        int i = blockIdx.x * blockDim.x + threadIdx.x;
        if (i < n) buf[i] += 1.0f;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int gen = g_gen;
            __threadfence();
            if (atomicAdd(&g_count, 1) == gridDim.x - 1) {
                g_count = 0;
                __threadfence();
                g_gen = gen + 1;
            } else {
                while (g_gen == gen) { }
            }
            __threadfence();
        }
        __syncthreads();
    }
}

template <int MODE>
float time_chain(float* buf, int n, int grid, int K, cudaStream_t s) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = 256;
        cfg.stream = s;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = a;
        cfg.numAttrs = MODE >= 1 ? 1 : 0;
        cudaLaunchKernelEx(&cfg, step_kernel<MODE>, buf, n);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    return ms * 1000.f / (10 * K);
}

int main() {
    const int K = 200;
    float* buf;
    const int nmax = 148 * 8 * 256;
    cudaMalloc(&buf, sizeof(float) * nmax);
    cudaMemset(buf, 0, sizeof(float) * nmax);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    int grids[] = {128, 148, 296, 977, 1184};
    for (int grid : grids) {
        const int n = grid * 256;
        printf("grid %5d: plain %.2f us  pdl-wait %.2f us  pdl-wait+trigger %.2f us per kernel\n", grid,
               time_chain<0>(buf, n, grid, K, s), time_chain<1>(buf, n, grid, K, s), time_chain<2>(buf, n, grid, K, s));
    }
    for (int grid : {148, 296}) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        persistent_kernel<<<grid, 256, 0, s>>>(buf, grid * 256, 10);
        cudaStreamSynchronize(s);
        cudaEventRecord(e0, s);
        persistent_kernel<<<grid, 256, 0, s>>>(buf, grid * 256, K);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("persistent grid %d: %.2f us per grid barrier\n", grid, ms * 1000.f / K);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
