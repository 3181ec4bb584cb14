// Latency floor probe: graph of R back-to-back launches of (a) an empty kernel, (b) a kernel
// streaming N bytes with 16-byte loads (one pass, all SMs), with and without PDL.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
__global__ void empty_k(int* p) { if (threadIdx.x == 12345) *p = 1; }
__global__ void stream_k(const uint4* __restrict__ src, size_t n16, int* out, int pdl) {
    if (pdl) { asm volatile("griddepcontrol.launch_dependents;"); asm volatile("griddepcontrol.wait;" ::: "memory"); }
    uint32_t x = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldg(src + i); x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (x == 0x12345678) *out = x;
}
int main() {
    const int R = 200;
    int* d; cudaMalloc(&d, 4);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // empty
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < R; ++i) empty_k<<<148, 128, 0, s>>>(d);
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEventRecord(e0, s); cudaGraphLaunch(ge, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); printf("empty kernel (148x128) in graph: %.2f us/launch\n", ms * 1000 / R);
    for (size_t mb : {1, 4, 16, 64}) {
        const int NB = 32;  // rotating buffers > L2 for the small sizes
        size_t bytes = mb << 20;
        std::vector<uint4*> bufs(NB);
        for (auto& b : bufs) { cudaMalloc(&b, bytes); cudaMemset(b, 1, bytes); }
        for (int pdl = 0; pdl < 2; ++pdl) for (int blocks : {148, 296, 592, 1184}) {
            cudaGraph_t g2; cudaGraphExec_t ge2;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < R; ++i) {
                cudaLaunchConfig_t cfg = {}; cfg.gridDim = blocks; cfg.blockDim = 256; cfg.stream = s;
                cudaLaunchAttribute at; at.id = cudaLaunchAttributeProgrammaticStreamSerialization; at.val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = &at; cfg.numAttrs = pdl;
                cudaLaunchKernelEx(&cfg, stream_k, (const uint4*)bufs[i % NB], bytes / 16, d, pdl);
            }
            cudaStreamEndCapture(s, &g2); cudaGraphInstantiate(&ge2, g2, 0);
            cudaGraphLaunch(ge2, s); cudaStreamSynchronize(s);
            cudaEventRecord(e0, s); cudaGraphLaunch(ge2, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double us = ms * 1000 / R;
            printf("stream %3zu MB blocks %4d pdl %d: %7.2f us/launch  %7.1f GB/s\n", mb, blocks, pdl, us, bytes / us / 1e3);
            cudaGraphExecDestroy(ge2); cudaGraphDestroy(g2);
        }
        for (auto& b : bufs) cudaFree(b);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
