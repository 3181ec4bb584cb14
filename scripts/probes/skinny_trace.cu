// Phase trace of the skinny exact kernel (skinny_mma_kernel) inside a CUDA graph of
// back-to-back launches, as bench.py runs it: per launch, %globaltimer stamps (thread 0 of
// every CTA) at entry, after the PDL wait, after the load+MMA loop, after the K reduction
// barrier and at exit.  Shows where a single skinny GEMM's microseconds go.
// Build + run on a B200:  bash scripts/probes/skinny_trace.sh
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int MAXL = 48, MAXCTA = 256;
__device__ unsigned long long g_st[MAXL][MAXCTA][5];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// The probe launches with gridDim.z = 1, so the kernel never uses batch_sc (it is multiplied by
// blockIdx.z = 0): the host passes the launch index there.  Plain per-CTA stores, no atomics,
// so the trace itself adds almost nothing to the kernel.
#define SKINNY_TRACE_AT(p) const unsigned long long _tr##p = (threadIdx.x == 0) ? gtime() : 0ull;
#define SKINNY_TRACE_END()                                                                        \
    if (threadIdx.x == 0 && batch_sc < MAXL && blockIdx.x < MAXCTA) {                             \
        unsigned long long* d_ = g_st[batch_sc][blockIdx.x];                                      \
        d_[0] = _tr0; d_[1] = _tr1; d_[2] = _tr2; d_[3] = _tr3; d_[4] = _tr4;                     \
    }

#include "../../paper_1910_00178_b200/csrc/kernel_skinny.cuh"

using ngemm_dev::skinny_mma_kernel;

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);       \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

template <int MT, int RG = 1>
void run(int m, int n, int k, int nbuf, int prefetch, int pdl, int ks_warps_log) {
    const int R = MAXL;
    std::vector<uint8_t*> as(nbuf), bs(nbuf);
    std::vector<int32_t*> cs(nbuf);
    for (int i = 0; i < nbuf; ++i) {
        CK(cudaMalloc(&as[i], (size_t)(m ? m : 1) * k));
        CK(cudaMalloc(&bs[i], (size_t)n * k));
        CK(cudaMalloc(&cs[i], (size_t)(m ? m : 1) * n * 4));
        CK(cudaMemset(as[i], 1, (size_t)(m ? m : 1) * k));
        CK(cudaMemset(bs[i], 1, (size_t)n * k));
    }
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int groups = (n + 16 * RG - 1) / (16 * RG);
    auto launch = [&](int i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(groups, 1, 1);
        cfg.blockDim = dim3(8 * 32);
        cfg.stream = s;
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at.val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = &at;
        cfg.numAttrs = pdl;
        const int vec = prefetch ? 3 : 1;
        CK(cudaLaunchKernelEx(&cfg, skinny_mma_kernel<MT, RG, 8>, (const uint8_t*)as[i % nbuf], (int64_t)k,
                              (const int8_t*)bs[i % nbuf], (int64_t)k, cs[i % nbuf], (int64_t)n, m, (int64_t)n,
                              (int64_t)k, (int64_t)k, vec, 0, (int64_t)0, (int64_t)0, (int64_t)i,
                              ngemm_dev::Requant()));
    };
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < R; ++i) launch(i);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaEventRecord(e1, s));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<unsigned long long> st((size_t)MAXL * MAXCTA * 5);
    CK(cudaMemcpyFromSymbol(st.data(), g_st, st.size() * 8));
    std::vector<unsigned long long> tr(MAXL * 5 * 2);
    for (int L = 0; L < R && L < MAXL; ++L)
        for (int p = 0; p < 5; ++p) {
            unsigned long long mn = ~0ull, mx = 0;
            for (int c = 0; c < groups && c < MAXCTA; ++c) {
                const unsigned long long v = st[((size_t)L * MAXCTA + c) * 5 + p];
                mn = v < mn ? v : mn;
                mx = v > mx ? v : mx;
            }
            tr[(L * 5 + p) * 2] = mn;
            tr[(L * 5 + p) * 2 + 1] = mx;
        }
    auto T = [&](int L, int p, int mx) { return (double)tr[(L * 5 + p) * 2 + mx]; };
    // average over launches 8..R-9 (steady state)
    double a[10] = {0};
    int cnt = 0;
    for (int L = 8; L < R - 8; ++L) {
        const double t0 = T(L, 0, 0);
        a[0] += T(L, 0, 1) - t0;                // entry spread (CTA launch)
        a[1] += T(L, 1, 0) - t0;                // first CTA released from the wait
        a[2] += T(L, 1, 1) - t0;                // last CTA released
        a[3] += T(L, 2, 0) - T(L, 1, 0);        // fastest load+MMA loop
        a[4] += T(L, 2, 1) - t0;                // last loop done
        a[5] += T(L, 3, 1) - t0;                // last reduction barrier
        a[6] += T(L, 4, 1) - t0;                // last exit
        a[7] += T(L + 1, 1, 0) - T(L, 4, 1);    // last exit -> next launch's first release
        a[8] += T(L + 1, 1, 0) - T(L, 1, 0);    // release-to-release period
        a[9] += T(L, 0, 0) - T(L - 1, 4, 1);    // this launch's first entry relative to the previous exit
        ++cnt;
    }
    for (double& x : a) x /= cnt;
    printf("RG%d %2dx%5dx%5d bufs=%2d pf=%d pdl=%d | %.2f us/launch | entry spread %.2f, wait release %.2f..%.2f, "
           "loop min %.2f, loops done %.2f, reduce %.2f, exit %.2f | exit->next release %.2f, period %.2f, "
           "entry-prev_exit %.2f (us)\n",
           RG, m, n, k, nbuf, prefetch, pdl, ms * 1000 / R, a[0] / 1e3, a[1] / 1e3, a[2] / 1e3, a[3] / 1e3, a[4] / 1e3,
           a[5] / 1e3, a[6] / 1e3, a[7] / 1e3, a[8] / 1e3, a[9] / 1e3);
    for (int i = 0; i < nbuf; ++i) {
        cudaFree(as[i]);
        cudaFree(bs[i]);
        cudaFree(cs[i]);
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(s);
}

int main(int argc, char** argv) {
    if (argc > 1) {  // focused mode: row groups per CTA (fewer, fatter CTAs co-reside with the previous grid)
        run<8, 1>(1, 4096, 1024, 64, 1, 1, 0);
        run<8, 2>(1, 4096, 1024, 64, 1, 1, 0);
        run<8, 4>(1, 4096, 1024, 64, 1, 1, 0);
        run<16, 1>(16, 4096, 1024, 64, 1, 1, 0);
        run<16, 2>(16, 4096, 1024, 64, 1, 1, 0);
        run<16, 4>(16, 4096, 1024, 64, 1, 1, 0);
        run<8, 1>(4, 3072, 768, 64, 1, 1, 0);
        run<8, 2>(4, 3072, 768, 64, 1, 1, 0);
        run<8, 1>(1, 768, 3072, 64, 1, 1, 0);
        run<8, 2>(1, 768, 3072, 64, 1, 1, 0);
        return 0;
    }
    for (int pdl = 1; pdl >= 0; --pdl)
        for (int pf = 1; pf >= 0; --pf)
            for (int nbuf : {1, 64}) {
                run<16>(16, 4096, 1024, nbuf, pf, pdl, 0);
                run<8>(1, 4096, 1024, nbuf, pf, pdl, 0);
                run<8>(1, 768, 768, nbuf, pf, pdl, 0);
                run<8>(4, 3072, 768, nbuf, pf, pdl, 0);
            }
    return 0;
}
