// D2H bandwidth of contiguous vs pitched (2D) copies into pinned host memory: 1 GiB of int32 C
// (16384 x 16384) copied as full rows, or as column tiles of 4096 / 8192 columns.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t n = 16384, bytes = n * n * 4;
    void *d, *h;
    cudaMalloc(&d, bytes);
    cudaMallocHost(&h, bytes);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (size_t tile : {n, n / 2, n / 4, n / 8}) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0, s);
            for (size_t c0 = 0; c0 < n; c0 += tile)
                for (size_t r0 = 0; r0 < n; r0 += 2048)
                    cudaMemcpy2DAsync((char*)h + (r0 * n + c0) * 4, n * 4, (char*)d + (r0 * n + c0) * 4, n * 4,
                                      tile * 4, 2048, cudaMemcpyDeviceToHost, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("D2H 1 GiB as %zu-column tiles (%zu B rows): %.2f ms, %.1f GiB/s\n", tile, tile * 4, ms,
                            1000.0 / ms);
        }
    }
    return 0;
}
