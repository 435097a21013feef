/*
 * apmm_cuda.h -- C ABI of the B200 (sm_100a) bipolar-INT arbitrary-precision matmul.
 *
 * This is the drop-in boundary for the reference's hot path (quantize -> bit-plane
 * decompose/pack -> WnAm matmul with shift-add recovery -> dequant). Every entry point
 * below names the reference C++ function it replaces (paths are relative to the
 * reference's proj/ directory). Plain pointers and sizes only; no C++ or torch types.
 *
 * Conventions
 *   - Return value: 0 (APMM_OK) on success, otherwise an apmm_status code. Codes 1..9
 *     map 1:1 onto the reference's apmm::Error subclasses (include/apmm/error.hpp:9-70);
 *     codes >= 100 are device-side failures the CPU reference cannot have.
 *   - Validation happens on the host BEFORE any device work, in the same order the
 *     reference checks (e.g. K agreement, then overflow_bound; kernel.cpp:189-199).
 *   - "Packed planes" always means the reference PackedBitPlanes buffer layout
 *     (include/apmm/bitplane.hpp:12-18): n planes, plane-major, then row, then
 *     ceil(cols/32) little-endian u32 words, column k at word k>>5 bit k&31, padding
 *     bits zero. Device entry points take that layout in device memory unchanged.
 *   - apmm_cu_* entry points take DEVICE pointers and are stream-ordered: they enqueue
 *     work on `stream` (NULL = the legacy default stream) and return without
 *     synchronising. Scratch comes from the
 *     context's workspace, grown on first use for a shape and reused afterwards.
 *   - apmm_* entry points without the cu_ prefix take HOST pointers and are
 *     synchronous (H2D, kernels, D2H on the context's stream). They are what a
 *     ctypes / cgo / JNI binding of the reference API calls.
 *   - A context is bound to one device and is not thread-safe; use one per thread.
 */
#ifndef APMM_CUDA_H_
#define APMM_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define APMM_API __attribute__((visibility("default")))
#else
#define APMM_API
#endif

typedef enum apmm_status {
  APMM_OK = 0,
  APMM_E_EVEN_VALUE = 1,          /* apmm::EvenValue         error.hpp:16-19 */
  APMM_E_OUT_OF_RANGE = 2,        /* apmm::OutOfRange        error.hpp:22-25 */
  APMM_E_NON_FINITE = 3,          /* apmm::NonFinite         error.hpp:28-31 */
  APMM_E_LENGTH_MISMATCH = 4,     /* apmm::LengthMismatch    error.hpp:34-37 */
  APMM_E_DIMENSION_MISMATCH = 5,  /* apmm::DimensionMismatch error.hpp:40-43 */
  APMM_E_INDEX_OUT_OF_BOUNDS = 6, /* apmm::IndexOutOfBounds  error.hpp:45-48 */
  APMM_E_OVERFLOW = 7,            /* apmm::Overflow          error.hpp:51-54 */
  APMM_E_OVERFLOW_BOUND = 8,      /* apmm::OverflowBound     error.hpp:57-60 */
  APMM_E_INVALID_ARGUMENT = 9,    /* null pointer / bad enum (reference: std::invalid_argument) */
  APMM_E_CUDA = 100,              /* CUDA runtime/driver error */
  APMM_E_NO_DEVICE = 101,         /* no usable device */
  APMM_E_UNSUPPORTED_DEVICE = 102 /* device is not sm_100 (B200) */
} apmm_status;

/* Granularity of quantization scales; bipolar.hpp:100-103. */
enum { APMM_PER_TENSOR = 0, APMM_PER_ROW = 1 };

typedef struct apmm_ctx apmm_ctx;
typedef struct CUstream_st* apmm_stream_t; /* == cudaStream_t */

/* ---- context ------------------------------------------------------------------- */
APMM_API int apmm_ctx_create(apmm_ctx** out, int device);
APMM_API int apmm_ctx_destroy(apmm_ctx* ctx);
/* Stream used by the synchronous host entry points (default: a private stream). */
APMM_API int apmm_ctx_set_stream(apmm_ctx* ctx, apmm_stream_t stream);
/* Human-readable message for the last failing call on this thread. */
APMM_API const char* apmm_last_error(void);
APMM_API const char* apmm_status_name(int status);
/* Library build/version string. */
APMM_API const char* apmm_version(void);
/* Number of kernel launches this context has enqueued (launch accounting for bench). */
APMM_API uint64_t apmm_ctx_launch_count(const apmm_ctx* ctx);

/* Kernel timing for measurement: when enabled, every launch of the given kernel class is
 * bracketed by CUDA events on the stream it is launched on. apmm_ctx_kernel_time
 * synchronises on those events and returns the summed device time (ms) and the number of
 * launches since the last reset, then resets. kernel: 0 = tensor-core GEMM (K3),
 * 1 = operand expansion (K1). */
APMM_API int apmm_ctx_enable_timing(apmm_ctx* ctx, int enable);
APMM_API int apmm_ctx_kernel_time(apmm_ctx* ctx, int kernel, double* total_ms, uint64_t* launches);

/* ---- scalar helpers (no device work) --------------------------------------------- */
/* overflow_bound (kernel.hpp:78-79, kernel.cpp:183-185): K*(2^n_w-1)*(2^n_x-1). */
APMM_API int apmm_overflow_bound(int n_w, int n_x, uint64_t k, int64_t* bound);
/* Words in a packed buffer: n * rows * ceil(cols/32) (bitplane.cpp:17-20). */
APMM_API uint64_t apmm_packed_words(int n, uint64_t rows, uint64_t cols);

/* ---- device entry points (stream-ordered, device pointers) ----------------------- */

/* decompose_and_pack (bitplane.hpp:49, bitplane.cpp:48-66): u8 codes [rows x cols]
 * (row-major, each < 2^n) -> packed planes. Codes >= 2^n are an OutOfRange on the
 * host API; here they are masked to n bits (the device cannot throw). */
APMM_API int apmm_cu_pack(apmm_ctx* ctx, const uint8_t* codes, uint64_t rows, uint64_t cols, int n,
                 uint32_t* planes, apmm_stream_t stream);

/* unpack (bitplane.hpp:52, bitplane.cpp:68-84): packed planes -> u8 codes. */
APMM_API int apmm_cu_unpack(apmm_ctx* ctx, const uint32_t* planes, uint64_t rows, uint64_t cols, int n,
                   uint8_t* codes, apmm_stream_t stream);

/* quantize + decompose_and_pack fused (bipolar.cpp:72-100 then bitplane.cpp:48-66):
 * fp64 values [rows x cols] -> packed planes + fp64 scales (1 for per-tensor, rows for
 * per-row). Arithmetic is IEEE fp64 exactly as the reference, so codes and scales are
 * bit-identical. `codes` may be NULL; when given it also receives the u8 codes.
 * Non-finite input is detected on device and reported as APMM_E_NON_FINITE after a
 * stream synchronisation (like apmm_cu_recover, a synchronising device entry point). */
APMM_API int apmm_cu_quantize_pack(apmm_ctx* ctx, const double* values, uint64_t rows, uint64_t cols,
                          int n, int granularity, uint32_t* planes, double* scales,
                          uint8_t* codes, apmm_stream_t stream);

/* matmul_ap (kernel.hpp:86-87, kernel.cpp:187-254): weights W [rows_w x k] at n_w bits,
 * features X [rows_x x k] at n_x bits (K-major), both packed planes ->
 * Y [rows_w x rows_x] int32 row-major, bit-exact with the reference for every input the
 * reference accepts. Rejects K*(2^n_w-1)*(2^n_x-1) > INT32_MAX with
 * APMM_E_OVERFLOW_BOUND before any device work. */
APMM_API int apmm_cu_matmul_ap(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                      const uint32_t* x_planes, uint64_t rows_x, int n_x, uint64_t k,
                      int32_t* y, apmm_stream_t stream);

/* matmul_ap followed by the CLI dequant epilogue (tools/apmm.cpp:329-340), fused:
 * out(m,n) = (float)((double)Y(m,n) * s_w(m) * s_x(n)), scales fp64 with per-tensor or
 * per-row granularity (a per-row X scale applies to output column n). The int32 product
 * never reaches HBM. */
APMM_API int apmm_cu_matmul_ap_dequant(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                              int n_w, const double* w_scales, int w_granularity,
                              const uint32_t* x_planes, uint64_t rows_x, int n_x,
                              const double* x_scales, int x_granularity, uint64_t k,
                              float* out, apmm_stream_t stream);

/* matmul_plane_pair (kernel.hpp:66-67, kernel.cpp:125-144): Y(m,n) = dot of weight plane
 * `weight_plane` row m with feature plane `feature_plane` row n, K - 2 popc(a ^ b), int32
 * [rows_w x rows_x]. Planes out of range -> APMM_E_INDEX_OUT_OF_BOUNDS; K > INT32_MAX ->
 * APMM_E_OVERFLOW_BOUND. Runs as a 1-bit x 1-bit matmul_ap on the plane slices. */
APMM_API int apmm_cu_matmul_plane_pair(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                              int n_w, int weight_plane, const uint32_t* x_planes,
                              uint64_t rows_x, int n_x, int feature_plane, uint64_t k,
                              int32_t* y, apmm_stream_t stream);

/* compute_plane_products (kernel.hpp:70-71, kernel.cpp:146-157): every plane pair,
 * stack[(i*n_x + j)][m][n] int32 (PlaneProductStack order, kernel.cpp:103-113). Debug /
 * property path: n_w*n_x GEMMs and an n_w*n_x x larger intermediate -- matmul_ap never forms
 * it. */
APMM_API int apmm_cu_compute_plane_products(apmm_ctx* ctx, const uint32_t* w_planes,
                                   uint64_t rows_w, int n_w, const uint32_t* x_planes,
                                   uint64_t rows_x, int n_x, uint64_t k, int32_t* stack,
                                   apmm_stream_t stream);

/* recover (kernel.hpp:74, kernel.cpp:159-181): y = sum_ij 2^(i+j) stack[i][j] in int64,
 * checked narrowing. Validates like the PlaneProductStack constructor: an entry outside
 * [-k, k] -> APMM_E_OUT_OF_RANGE (kernel.cpp:91-101); a result outside int32 ->
 * APMM_E_OVERFLOW. Synchronises the stream to report those. */
APMM_API int apmm_cu_recover(apmm_ctx* ctx, const int32_t* stack, int n_w, int n_x, uint64_t k,
                    uint64_t rows, uint64_t cols, int32_t* y, apmm_stream_t stream);

/* The reference flow quantize(X) -> decompose_and_pack -> matmul_ap -> dequant
 * (tools/apmm.cpp:275-340, bipolar.cpp:72-100) with the feature quantizer writing the GEMM's
 * u8 operand directly (no feature planes, no feature expansion):
 * fp64 X [rows_x x k] -> x_scales (device, 1 or rows_x doubles) and
 * out = (float)((double)Y * s_w * s_x) [rows_w x rows_x]. Bit-identical to
 * apmm_cu_quantize_pack followed by apmm_cu_matmul_ap_dequant. Synchronises the stream
 * once (after the quantizer) to report APMM_E_NON_FINITE before the overflow_bound check
 * and the GEMM, in the reference's order. */
APMM_API int apmm_cu_quantize_matmul_ap_dequant(apmm_ctx* ctx, const uint32_t* w_planes,
                                       uint64_t rows_w, int n_w, const double* w_scales,
                                       int w_granularity, const double* x_values,
                                       uint64_t rows_x, uint64_t k, int n_x, int x_granularity,
                                       double* x_scales, float* out, apmm_stream_t stream);

/* ---- host entry points (synchronous, host pointers) ------------------------------- */
/* These mirror the reference functions one for one and add the H2D/D2H copies. */

/* decompose_and_pack (bitplane.cpp:48-66). Validates codes < 2^n -> OutOfRange, as the
 * CodeMatrix constructor does (bipolar.cpp:33-36). */
APMM_API int apmm_decompose_and_pack(apmm_ctx* ctx, const uint8_t* codes, uint64_t rows, uint64_t cols,
                            int n, uint32_t* planes);

/* unpack (bitplane.cpp:68-84). Validates zero padding like the PackedBitPlanes
 * constructor (bitplane.cpp:22-32). */
APMM_API int apmm_unpack(apmm_ctx* ctx, const uint32_t* planes, uint64_t rows, uint64_t cols, int n,
                uint8_t* codes);

/* quantize (bipolar.cpp:72-100) + decompose_and_pack: codes (may be NULL), planes,
 * scales (1 or rows doubles). */
APMM_API int apmm_quantize_pack(apmm_ctx* ctx, const double* values, uint64_t rows, uint64_t cols,
                       int n, int granularity, uint8_t* codes, uint32_t* planes,
                       double* scales);

/* compute_plane_products (kernel.cpp:146-157) with host buffers; validates padding. */
APMM_API int apmm_compute_plane_products(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                                int n_w, const uint32_t* x_planes, uint64_t rows_x, int n_x,
                                uint64_t k, int32_t* stack);

/* recover (kernel.cpp:159-181) with host buffers. */
APMM_API int apmm_recover(apmm_ctx* ctx, const int32_t* stack, int n_w, int n_x, uint64_t k,
                 uint64_t rows, uint64_t cols, int32_t* y);

/* matmul_ap (kernel.cpp:187-254). Validates padding like PackedBitPlanes
 * (bitplane.cpp:22-32), then K agreement and overflow_bound like kernel.cpp:189-199. */
APMM_API int apmm_matmul_ap(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                   const uint32_t* x_planes, uint64_t rows_x, int n_x, uint64_t k, int32_t* y);

/* matmul_ap + dequant epilogue (tools/apmm.cpp:322-340) -> float [rows_w x rows_x]. */
APMM_API int apmm_matmul_ap_dequant(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                           const double* w_scales, int w_granularity, const uint32_t* x_planes,
                           uint64_t rows_x, int n_x, const double* x_scales,
                           int x_granularity, uint64_t k, float* out);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* APMM_CUDA_H_ */
