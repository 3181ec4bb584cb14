/*
 * ngemm_cuda.h — the C-ABI drop-in boundary of the B200 u8 x i8 -> i32 GEMM engine
 * (libngemm_cuda.so, hand-written sm_100a CUDA; no CPU fallback, no CUTLASS/cuBLAS).
 *
 * Plain pointers, sizes and status codes only.  Each entry point names the reference
 * interface it replaces (paths under /root/reference/proj/include/ngemm):
 *
 *   reference                                                      -> this ABI
 *   native::avx*_conv_u8i8_sat(a, b, c, m, n, k)                   -> ngemm_cuda_gemm_u8i8
 *        (simd_native.hpp:144-147, 215-218; gemm.hpp:336-350)
 *   native::avx*_ngemm_u8i8_sat(PackedWeight&, MatrixBuf&, C&)     -> ngemm_cuda_packed_upload +
 *        (simd_native.hpp:282-283, 361-363; gemm.hpp:385-395)          ngemm_cuda_gemm_packed
 *   detail::emu_conv_u8i8 / emu_ngemm_u8i8 (Engine::Emulated)       -> kernel NGEMM_KERNEL_SIMT
 *        (gemm.hpp:113-159, 192-243)
 *   gemm_conventional / gemm_ngemm on host MatrixBufs               -> ngemm_cuda_gemm_u8i8_host /
 *        (gemm.hpp:327-369, 373-409)                                   ngemm_cuda_gemm_packed_host
 *   PackedWeight::block_offset inverse (layout.hpp:152-171)         -> ngemm_cuda_repack
 *
 * Semantics (bit-exact):
 *   sat_mode 1 (WideningExact):      C[m][n] = sum_k A[m][k]*B[n][k]  mod 2^32   (gemm.hpp:36-52)
 *   sat_mode 0 (HardwareSaturating): C[m][n] = sum_j sat16(A[m][2j]B[n][2j] + A[m][2j+1]B[n][2j+1])
 *                                    mod 2^32, odd K tail paired with 0     (gemm.hpp:83-104)
 *   (0/1 follow the reference enum order, lanes.hpp:18.)
 *
 * Conventions: A is [M x K] u8 row-major (row stride lda bytes), B is [N x K] i8 row-major
 * (ldb), C is [M x N] i32 row-major (ldc elements).  C is fully overwritten (no zero-init
 * needed).  Errors are reported before any launch and map 1:1 to the reference exception
 * types (common.hpp:77-127).  Device-pointer entries are asynchronous on `stream`
 * (a cudaStream_t, NULL = legacy default stream) and reentrant per stream.
 */
#ifndef NGEMM_CUDA_H
#define NGEMM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NGEMM_CUDA_ABI_VERSION 1

typedef enum {
    NGEMM_OK = 0,
    NGEMM_ERR_SHAPE = 1,       /* ShapeError        (common.hpp:82-85) */
    NGEMM_ERR_UNSUPPORTED = 2, /* UnsupportedError  (common.hpp:114-117) */
    NGEMM_ERR_CONFIG = 3,      /* ConfigError       (common.hpp:104-107) */
    NGEMM_ERR_RANGE = 4,       /* RangeError        (common.hpp:87-90) */
    NGEMM_ERR_CORRUPTION = 5,  /* CorruptionError   (common.hpp:109-112) */
    NGEMM_ERR_INDEX = 6,       /* IndexError        (common.hpp:92-95) */
    NGEMM_ERR_CUDA = 7,        /* CUDA runtime failure (Error base class) */
    NGEMM_ERR_TUNE = 8         /* TuneError         (common.hpp:124-127) */
} ngemm_status;

typedef enum {
    NGEMM_SAT_HARDWARE = 0, /* SatMode::HardwareSaturating */
    NGEMM_SAT_EXACT = 1     /* SatMode::WideningExact */
} ngemm_sat_mode;

/* Kernel selection; AUTO is what every reference-facing entry uses. */
typedef enum {
    NGEMM_KERNEL_AUTO = 0,
    NGEMM_KERNEL_TCGEN05 = 1, /* tensor-core tcgen05.mma kind::i8 (exact mode only; AUTO runs the
                                 saturating mode on it too, for the pairs that cannot clamp) */
    NGEMM_KERNEL_SIMT = 2,    /* CUDA-core dp4a tiled kernel, both modes (the Engine::Emulated path) */
    NGEMM_KERNEL_SKINNY = 3,  /* memory-bound M <= 16 path, both modes */
    NGEMM_KERNEL_SAT_HYBRID = 4 /* HardwareSaturating only, M > 16, C 16-byte aligned with ldc % 4 == 0:
                                   tcgen05 on the pairs that cannot clamp + CUDA-core fix of the rest
                                   (AUTO picks it for M >= 256 and >= 1e9 MACs) */
} ngemm_kernel;

/* PackedWeight metadata (layout.hpp:120-135; NGPT trailer layout.hpp:283-293).  h = 4 is the
 * u8 path (1-byte elements), h = 2 the i16 path (2-byte elements); packed byte size is
 * m_pad * k_pad * element size. */
typedef struct {
    int32_t w, h, v;      /* KernelShape */
    int64_t tm, tn, tk;   /* TileConfig */
    int32_t perm;         /* Perm tag 0..5 = MNK MKN NMK NKM KMN KNM (layout.hpp:54) */
    int64_t m_orig, k_orig;
    int64_t m_pad, k_pad; /* must equal round_up(m_orig, tm), round_up(k_orig, tk) */
} ngemm_packed_meta;

/* Opaque device-resident prepacked weight: the K-major, 16-byte-stride copy of A that the
 * kernels consume, made once per weight (the paper's offline prepack). */
typedef struct ngemm_packed_dev* ngemm_packed_handle;

/* ---- device-pointer entries ------------------------------------------------------------ */

/* C = A * B^T on device pointers (replaces avx*_conv_u8i8_sat). */
ngemm_status ngemm_cuda_gemm_u8i8(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                                  int32_t* c, int64_t ldc, int64_t m, int64_t n, int64_t k,
                                  int sat_mode, void* stream);

/* A strided batch of `batch` independent GEMMs of one shape: operand z of A / B / C starts at
 * a + z*stride_a, b + z*stride_b, c + z*stride_c (element strides; 0 on A or B broadcasts that
 * operand; C slices must not overlap).  The reference has no batched entry — its callers loop
 * over gemm_conventional (gemm.hpp:327-369) once per request; for the skinny (M <= 16)
 * serving shapes this issues one launch for the whole batch instead. */
ngemm_status ngemm_cuda_gemm_u8i8_strided_batched(const uint8_t* a, int64_t lda, int64_t stride_a,
                                                  const int8_t* b, int64_t ldb, int64_t stride_b,
                                                  int32_t* c, int64_t ldc, int64_t stride_c,
                                                  int64_t batch, int64_t m, int64_t n, int64_t k,
                                                  int sat_mode, void* stream);

/* GEMM with a fused requantisation epilogue (the paper's "operation fusion" extension,
 * PAPER.md:422-423; no reference counterpart): int8 out[M x N] (row stride ldo) with
 *   out[r][c] = clamp(rint(float(C[r][c] + bias[c]) * scale[c]) + zero_point, -128, 127)
 * where C is the int32 GEMM of sat_mode, the int32 + bias add wraps, float(.) rounds to nearest,
 * the product is one IEEE fp32 multiply and rint rounds half to even.  scale: N floats (device),
 * bias: N int32 (device) or NULL.  Exact mode requantises in the kernel's epilogue (tcgen05 for
 * M > 16, the warp-MMA stream for M <= 16; int32 C is never written to memory); the saturating
 * mode computes C in scratch and requantises it. */
ngemm_status ngemm_cuda_gemm_u8i8_requant(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                                          int8_t* out, int64_t ldo, int64_t m, int64_t n, int64_t k,
                                          const float* scale, const int32_t* bias, int zero_point,
                                          int sat_mode, void* stream);

/* Same, forcing one kernel (tests / bench / ncu evidence per kernel choice). */
ngemm_status ngemm_cuda_gemm_u8i8_ex(const uint8_t* a, int64_t lda, const int8_t* b, int64_t ldb,
                                     int32_t* c, int64_t ldc, int64_t m, int64_t n, int64_t k,
                                     int sat_mode, int kernel, void* stream);

/* Device repack: packed bytes (d_packed, m_pad*k_pad) -> row-major A (m_orig x k_orig, row
 * stride lda >= k_orig) on `stream`.  Inverse of PackedWeight::elem_offset. */
ngemm_status ngemm_cuda_repack(const ngemm_packed_meta* meta, const uint8_t* d_packed, uint8_t* d_a,
                               int64_t lda, void* stream);

/* Validates the metadata like TileConfig::validate / pack_weights (layout.hpp:92-102, 258-263). */
ngemm_status ngemm_cuda_packed_validate(const ngemm_packed_meta* meta);

/* Upload host packed bytes to the current device and repack to the device-resident layout. */
ngemm_status ngemm_cuda_packed_upload(const ngemm_packed_meta* meta, const uint8_t* host_packed,
                                      size_t nbytes, ngemm_packed_handle* out);
/* Build a handle from an already device-resident row-major A (device copy is made). */
ngemm_status ngemm_cuda_packed_from_device(const uint8_t* d_a, int64_t lda, int64_t m, int64_t k,
                                           ngemm_packed_handle* out);
ngemm_status ngemm_cuda_packed_free(ngemm_packed_handle h);
/* Device pointer / row stride of the handle's K-major A (for custom launches). */
ngemm_status ngemm_cuda_packed_info(ngemm_packed_handle h, const uint8_t** d_a, int64_t* lda,
                                    int64_t* m, int64_t* k, int* device);

/* C = unpack(P) * B^T with a device-resident handle (replaces avx*_ngemm_u8i8_sat). */
ngemm_status ngemm_cuda_gemm_packed(ngemm_packed_handle h, const int8_t* b, int64_t ldb, int32_t* c,
                                    int64_t ldc, int64_t n, int sat_mode, void* stream);

/* ---- host-pointer entries (synchronous; what the C++ drop-in headers call) -------------- */

ngemm_status ngemm_cuda_gemm_u8i8_host(const uint8_t* a, const int8_t* b, int32_t* c, int64_t m,
                                       int64_t n, int64_t k, int sat_mode, int kernel);
/* Packed weight + input, host pointers; the weight kind follows meta->h (4: u8 weight with i8 b,
 * 2: i16 weight with i16 b; the 16-bit path has no saturation stage, gemm.hpp:161-190). */
ngemm_status ngemm_cuda_gemm_packed_host(const ngemm_packed_meta* meta, const uint8_t* host_packed,
                                         size_t nbytes, const void* b, int32_t* c, int64_t n,
                                         int sat_mode, int kernel);

/* Device-resident weight handle + HOST input B and output C (what gemm_ngemm calls: the weight
 * stays on the device across calls, B and C cross the bus per call). */
ngemm_status ngemm_cuda_gemm_packed_resident_host(ngemm_packed_handle h, const int8_t* b, int32_t* c,
                                                  int64_t n, int sat_mode);

/* ---- the reference's 16-bit path: i16 x i16 -> i32 (gemm.hpp:161-190, 245-281;
 * madd_pair_i16 wraps mod 2^32, lanes.hpp:42-47).  CUDA-core kernel; lda/ldb in elements. */
ngemm_status ngemm_cuda_gemm_i16(const int16_t* a, int64_t lda, const int16_t* b, int64_t ldb, int32_t* c,
                                 int64_t ldc, int64_t m, int64_t n, int64_t k, void* stream);
ngemm_status ngemm_cuda_gemm_i16_host(const int16_t* a, const int16_t* b, int32_t* c, int64_t m, int64_t n,
                                      int64_t k);
ngemm_status ngemm_cuda_gemm_packed_i16(ngemm_packed_handle h, const int16_t* b, int64_t ldb, int32_t* c,
                                        int64_t ldc, int64_t n, void* stream);

/* ---- multi-GPU M-shard driver (single process, one stream per device) -------------------
 * A's rows are split into ndev contiguous, tile-aligned blocks; B is replicated; device d
 * writes rows [row_start[d], row_start[d+1]) of C.  Host pointers; if gather_device >= 0
 * the full C is also assembled on that device (peer copies over NVLink) and returned in
 * *gathered (caller frees with ngemm_cuda_free). */
ngemm_status ngemm_cuda_shard_rows(int64_t m, int ndev, int64_t align, int64_t* row_start /* ndev+1 */);
ngemm_status ngemm_cuda_gemm_u8i8_multi(const int* devices, int ndev, const uint8_t* a, const int8_t* b,
                                        int32_t* c, int64_t m, int64_t n, int64_t k, int sat_mode,
                                        int gather_device, int32_t** gathered);
ngemm_status ngemm_cuda_free(void* device_ptr);
/* The multi-GPU driver enables peer access between the listed devices, copies B over PCIe ONCE
 * (into devices[0]) and relays it device to device over NVLink in 16 MiB chunks; each device
 * then streams its A rows in and its C rows out through the host pipeline (pinned or pageable
 * host buffers), and with a gather also peer-copies its C rows into the gather buffer. */

/* Sharded resident weight (gemm_ngemm over several GPUs, layout.hpp:159-161): the packed rows
 * are split into tile-aligned blocks of whole tm-strips (ngemm_cuda_shard_rows, align =
 * lcm(tm, 128)); out[d] receives the handle of device devices[d] (NULL when that device gets no
 * rows).  Free each with ngemm_cuda_packed_free.  u8 weights. */
ngemm_status ngemm_cuda_packed_upload_sharded(const ngemm_packed_meta* meta, const uint8_t* host_packed,
                                              size_t nbytes, const int* devices, int ndev,
                                              ngemm_packed_handle* out /* ndev */);
/* C[M x N] (host) = the sharded weight x B^T: B replicated by one H2D + NVLink relay, each device
 * computes its row block from its resident shard. */
ngemm_status ngemm_cuda_gemm_packed_multi(const ngemm_packed_handle* shards, int ndev, const int8_t* b,
                                          int32_t* c, int64_t n, int sat_mode);

/* ---- GPU autotuner (replaces the CPU tile search of tuner.hpp:132-245) -------------------- */
typedef struct {
    int64_t m, n, k;
    int32_t sat_mode;
    int32_t kernel;          /* NGEMM_KERNEL_* that won */
    int32_t tc_cfg;          /* tcgen05 tile configuration (-1 = not applicable) */
    int32_t tc_splits;       /* tcgen05 split-K factor (-1 = not applicable) */
    int32_t skinny_variant;  /* skinny kernel variant (-1 = not applicable) */
    double median_ns, min_ns;
    int32_t trials;
    int64_t timestamp;       /* seconds since the epoch */
} ngemm_tune_record;

/* Times every applicable kernel configuration for (m, n, k, sat_mode) on the current device
 * (seeded full-range operands), verifying each bit-for-bit against the CUDA-core reference
 * kernel before its timing counts (NGEMM_ERR_TUNE on a mismatch); the fastest becomes the
 * dispatcher's choice for that shape in this process.  repeats >= 3, warmup >= 1. */
ngemm_status ngemm_cuda_tune(int64_t m, int64_t n, int64_t k, int sat_mode, int repeats, int warmup,
                             ngemm_tune_record* out);
/* Append-only text store, one record per line, last record for a shape wins. */
ngemm_status ngemm_cuda_tune_store_save(const char* path);
ngemm_status ngemm_cuda_tune_store_load(const char* path, int* loaded);
ngemm_status ngemm_cuda_tune_clear(void);

/* ---- experiment / test knobs and the scratch pool ---------------------------------------
 * Kernel-selection overrides used by the tests and sweep scripts (never needed in production):
 * PDL, L2_PREFETCH, SKINNY_FAST, SKINNY_SPLITS, SKINNY_RG, SKINNY_WARPS, SKINNY_VARIANT, TC_QUAD,
 * TC_CFG, TC_SPLITS, TC_DIRECT, TC_PREISSUE, TC_L2HINT, TC_GROUP_M, TC_DBG, SAT_HYBRID,
 * SATFIX_SKIP, I16_PATH (1 tcgen05 / 0 simt), REQUANT_UNFUSED, TC_SCHED; -1 = unset.  Initial
 * values are read ONCE from NGEMM_<NAME> environment variables; the launch path never reads the
 * environment.  Names may carry the NGEMM_ prefix.  get_option returns INT32_MIN for an unknown
 * name; reset_options re-reads the environment. */
ngemm_status ngemm_cuda_set_option(const char* name, int value);
int ngemm_cuda_get_option(const char* name);
ngemm_status ngemm_cuda_reset_options(void);
/* Scratch buffers come from a private stream-ordered pool per device (the device's default pool
 * is never reconfigured); trim returns the current device's cached scratch to the driver. */
ngemm_status ngemm_cuda_trim(void);

/* ---- introspection ----------------------------------------------------------------------- */
/* Current CUDA device of the calling thread. */
ngemm_status ngemm_cuda_device(int* device);
int ngemm_cuda_abi_version(void);
const char* ngemm_cuda_status_name(int status);
/* Thread-local message of the last failing call on this thread ("" if none). */
const char* ngemm_cuda_last_error(void);
/* Kernel AUTO would pick for a shape (NGEMM_KERNEL_*), without launching. */
int ngemm_cuda_pick_kernel(int64_t m, int64_t n, int64_t k, int sat_mode);
/* Number of kernels this library launched since load (all entries, all threads). */
uint64_t ngemm_cuda_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* NGEMM_CUDA_H */
