// Cost of per-CTA same-address atomics at the end of a 977-CTA kernel (B200):
// (0) none, (1) one fp64 atomicAdd (RED) per CTA, (2) last-CTA counter (atomicAdd with
// return + __threadfence), (3) both, (4) per-CTA partials + last-CTA sum.  Graph of K launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/atomics tools/ubench/atomics.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ double g_sum;
__device__ unsigned g_ctr;
__device__ double g_part[4096];

template <int MODE>
__global__ void k(float* buf, int n) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    float v = 0.f;
    if (i < n) { v = buf[i]; buf[i] = v + 1.0f; }
    __shared__ double red[8];
    __shared__ int last;
    double b = v;
    for (int o = 16; o; o >>= 1) b += __shfl_xor_sync(0xffffffff, b, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = b;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0; for (int w = 0; w < 8; ++w) s += red[w];
        if (MODE == 1 || MODE == 3) atomicAdd(&g_sum, s);
        red[0] = s;
        if (MODE == 4) g_part[blockIdx.x] = s;
        if (MODE >= 2) {
            __threadfence();
            const unsigned prev = atomicAdd(&g_ctr, 1u);
            last = prev == gridDim.x - 1;
        }
    }
    if (MODE == 5 || MODE == 6) {             // 51 per-CTA column atomics
        __syncthreads();
        if (threadIdx.x < 51) atomicAdd(&g_part[MODE == 5 ? threadIdx.x : threadIdx.x * 32], red[0]);
        return;
    }
    if (MODE >= 2) {
        __syncthreads();
        if (last) {
            if (MODE == 4) {
                __threadfence();
                double s = 0;
                for (int c = threadIdx.x; c < gridDim.x; c += blockDim.x) s += ((volatile double*)g_part)[c];
                for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
                if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
                __syncthreads();
                if (threadIdx.x == 0) { double t = 0; for (int w = 0; w < 8; ++w) t += red[w]; g_sum = t; }
            }
            if (threadIdx.x == 0) g_ctr = 0;
        }
    }
}

template <int MODE>
float run(float* buf, int grid, int K, cudaStream_t s) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < K; ++i) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = grid; cfg.blockDim = 256; cfg.stream = s;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = a; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k<MODE>, buf, grid * 256);
    }
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1000.f / (10 * K);
}

int main() {
    float* buf; cudaMalloc(&buf, sizeof(float) * 4096 * 256); cudaMemset(buf, 0, sizeof(float) * 4096 * 256);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int grid : {148, 977, 2048}) {
        printf("grid %4d: none %.2f  red %.2f  lastcta %.2f  both %.2f  partials+lastcta %.2f  51 consecutive %.2f  51 strided %.2f us/kernel\n", grid,
               run<0>(buf, grid, 200, s), run<1>(buf, grid, 200, s), run<2>(buf, grid, 200, s),
               run<3>(buf, grid, 200, s), run<4>(buf, grid, 200, s), run<5>(buf, grid, 200, s), run<6>(buf, grid, 200, s));
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
