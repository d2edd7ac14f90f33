#include <cuda_runtime.h>
#include <cstdio>
__global__ void step(int* ctr, int k, cudaGraphConditionalHandle h) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int j = ++ctr[0];
        if (j >= k) cudaGraphSetConditional(h, 0);
    }
}
__global__ void work(float* b, int n) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) b[i] += 1.f;
}
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    int* ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
    float* b; cudaMalloc(&b, 4 << 20); cudaMemset(b, 0, 4 << 20);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
    printf("add node: %s\n", cudaGetErrorString(e));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    printf("begin capture: %s\n", cudaGetErrorString(e));
    for (int r = 0; r < 3; ++r) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = 977; cfg.blockDim = 256; cfg.stream = s;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = a; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, work, b, 977 * 256);
    }
    {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = 1; cfg.blockDim = 32; cfg.stream = s;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        a[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = a; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, step, ctr, 100, h);
    }
    e = cudaStreamEndCapture(s, &body);
    printf("end capture: %s\n", cudaGetErrorString(e));
    cudaGraphExec_t ge;
    e = cudaGraphInstantiate(&ge, g, 0);
    printf("instantiate: %s\n", cudaGetErrorString(e));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaMemset(ctr, 0, 4);
    cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int hc; cudaMemcpy(&hc, ctr, 4, cudaMemcpyDeviceToHost);
    printf("iterations %d, %.2f us per iteration (4 kernels), err %s\n", hc, ms * 1000 / hc, cudaGetErrorString(cudaGetLastError()));
}
