// What sets the PDL release latency between back-to-back launches?  Minimal kernels (148 CTAs x
// 256 threads, graph of 48 launches, programmatic stream serialization) that add one feature
// of the tcgen05 GEMM kernel at a time; prints the average time from the last CTA exit of
// launch L to the first griddepcontrol.wait return in launch L+1, and us per launch.
// Build + run on a B200:  bash scripts/probes/pdl_gap.sh
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

constexpr int R = 48, NCTA = 148;
__device__ unsigned long long g_rel[R][NCTA], g_exit[R][NCTA];

__device__ __forceinline__ unsigned long long now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// feature bits: 1 = touch 200 KB dynamic smem, 2 = TMEM alloc/dealloc (512 cols),
// 4 = + relinquish_alloc_permit, 8 = one 4 KB bulk store smem->global + wait, 16 = mbarrier init,
// 32 = launch_dependents at the start (else implicit at exit)
struct alignas(64) BigParam {
    uint8_t bytes[384];  // three CUtensorMaps' worth of __grid_constant__ kernel parameters
};

// 64 = cluster launch attribute (dims 1), 128 = cluster dims 2, 256 = 384 B of grid-constant params,
// 512 = one TMA 2D tensor load (128 x 128 bytes) completed on an mbarrier, 1024 = prefetch.tensormap,
// 2048 = tcgen05.ld of 32 columns (with bit 2)
template <int F>
__global__ void __launch_bounds__(256, 1) probe_k(int launch, int* out, const __grid_constant__ BigParam bp,
                                                  const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    if (F & 32) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (F & 16) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
    }
    if (F & 2) {
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&tslot)));
            if (F & 4) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    if ((F & 1024) && threadIdx.x == 0)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) g_rel[launch][blockIdx.x] = now();
    if (F & 512) {
        const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
        if (threadIdx.x == 0) {
            if (!(F & 16)) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(16384) : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(smem)),
                "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(0), "r"((int)(blockIdx.x % 8) * 128), "r"(b)
                : "memory");
            asm volatile(
                "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b)
                : "memory");
        }
    }
    if ((F & 2048) && (F & 2) && threadIdx.x < 128) {
        uint32_t v[32];
        const uint32_t taddr = tslot + ((threadIdx.x / 32 * 32) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
              "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
              "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t x = 0;
        for (int i = 0; i < 32; ++i) x ^= v[i];
        if (x == 0x12345678u) out[1] = 1;
    }
    if (F & 1) {
        for (int i = threadIdx.x; i < 200 * 1024 / 16; i += 256) reinterpret_cast<uint4*>(smem)[i] = make_uint4(i, 0, 0, 0);
    }
    __syncthreads();
    if (F & 8) {
        if (threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(
                             out + blockIdx.x * 1024),
                         "r"((uint32_t)__cvta_generic_to_shared(smem))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
    }
    __syncthreads();
    if (F & 2) {
        if (threadIdx.x < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
    }
    __syncthreads();
    if ((F & 256) && bp.bytes[threadIdx.x] == 255) out[0] = 1;
    if (threadIdx.x == 0) g_exit[launch][blockIdx.x] = now();
}

#define CK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) {                                                                  \
            printf("CUDA error %s at line %d\n", cudaGetErrorString(e_), __LINE__);               \
            exit(1);                                                                              \
        }                                                                                         \
    } while (0)

CUtensorMap g_map;

template <int F>
void run(const char* name, int* out) {
    const int smem = (F & 1) ? 200 * 1024 : ((F & (8 | 512)) ? 16384 + 1024 : 0);
    CK(cudaFuncSetAttribute(probe_k<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < R; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(NCTA);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = (F & 128) ? 2 : 1;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = (F & (64 | 128)) ? 2 : 1;
        BigParam bp{};
        CK(cudaLaunchKernelEx(&cfg, probe_k<F>, i, out, bp, g_map));
    }
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
    std::vector<unsigned long long> rel(R * NCTA), ex(R * NCTA);
    CK(cudaMemcpyFromSymbol(rel.data(), g_rel, rel.size() * 8));
    CK(cudaMemcpyFromSymbol(ex.data(), g_exit, ex.size() * 8));
    double gap = 0, body = 0;
    int n = 0;
    for (int L = 4; L < R - 1; ++L) {
        unsigned long long mx = 0, mn_next = ~0ull, mn_rel = ~0ull;
        for (int c = 0; c < NCTA; ++c) {
            mx = ex[L * NCTA + c] > mx ? ex[L * NCTA + c] : mx;
            mn_next = rel[(L + 1) * NCTA + c] < mn_next ? rel[(L + 1) * NCTA + c] : mn_next;
            mn_rel = rel[L * NCTA + c] < mn_rel ? rel[L * NCTA + c] : mn_rel;
        }
        gap += (double)(mn_next - mx);
        body += (double)(mx - mn_rel);
        ++n;
    }
    printf("%-44s %6.2f us/launch | release->last exit %5.2f us | last exit->next release %5.2f us\n", name,
           ms * 1000 / R, body / n / 1e3, gap / n / 1e3);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(s);
}

int main() {
    int* out;
    CK(cudaMalloc(&out, NCTA * 4096));
    uint8_t* src;
    CK(cudaMalloc(&src, 1024 * 1024));
    {
        using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        cuuint64_t dims[2] = {1024, 1024}, strides[1] = {1024};
        cuuint32_t box[2] = {128, 128}, es[2] = {1, 1};
        CUresult r = reinterpret_cast<EncFn>(fn)(&g_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, dims, strides, box, es,
                                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    }
    run<0>("plain (implicit trigger)", out);
    run<32>("launch_dependents at start", out);
    run<32 | 1>("+ 200 KB dynamic smem", out);
    run<32 | 16>("+ mbarrier init", out);
    run<32 | 8>("+ bulk store + wait_group 0", out);
    run<32 | 2>("+ TMEM alloc/dealloc", out);
    run<32 | 2 | 4>("+ TMEM alloc/relinquish/dealloc", out);
    run<32 | 1 | 2 | 8 | 16>("all but relinquish", out);
    run<32 | 64>("cluster attribute, dims 1", out);
    run<32 | 128>("cluster dims 2", out);
    run<32 | 256>("384 B grid-constant params (used)", out);
    run<32 | 512>("TMA tensor load + mbarrier wait", out);
    run<32 | 1024>("prefetch.tensormap", out);
    run<32 | 512 | 1024>("TMA load + prefetch.tensormap", out);
    run<32 | 2 | 2048>("TMEM alloc + tcgen05.ld", out);
    run<32 | 2 | 16 | 512 | 1024 | 2048>("TMA + TMEM + tcgen05.ld + mbarrier", out);
    return 0;
}
