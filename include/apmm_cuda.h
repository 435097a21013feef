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
 *     synchronising. Scratch comes from the context's workspace, grown (stream-ordered,
 *     never with a device-wide synchronisation) on first use for a larger shape and reused
 *     afterwards; apmm_ctx_reserve pre-sizes it. Growth is impossible while `stream` is
 *     being captured into a CUDA graph: such a call fails with APMM_E_INVALID_ARGUMENT
 *     and the caller reserves first.
 *   - apmm_* entry points without the cu_ prefix take HOST pointers and are
 *     synchronous (H2D, kernels, D2H on the context's stream). They are what a
 *     ctypes / cgo / JNI binding of the reference API calls.
 *   - One context = one device, one stream, one thread. The workspace is not tied to a
 *     stream by CUDA, so the context binds itself to the stream of its first device call
 *     (or the one given to apmm_ctx_set_stream); a device call on any other stream fails
 *     with APMM_E_INVALID_ARGUMENT instead of racing on the workspace. Use one context
 *     per stream for concurrency. The bound stream must outlive its binding.
 *   - Programmatic dependent launch: consecutive calls on the bound stream overlap (the
 *     next call's weight expansion runs while the previous GEMM drains). Only WEIGHT
 *     planes are read before the previous kernel in the stream has completed; feature
 *     planes, scales and outputs are touched only after it. Weights therefore must not
 *     be written by a kernel that triggers its dependents early
 *     (griddepcontrol.launch_dependents) and is launched immediately before the call;
 *     uploads (cudaMemcpy*) and ordinary kernels are always safe.
 *     apmm_ctx_set_option(APMM_OPT_EARLY_WEIGHT_READ, 0) turns the early read off.
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
  APMM_E_PARSE = 10,              /* apmm::ParseError        error.hpp:62-65 */
  APMM_E_IO = 11,                 /* apmm::IoError           error.hpp:67-70 */
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
/* Bind the context to `stream`: the host entry points run on it and the device entry points
 * must be given it (default: a private stream for the host entry points, and the stream of
 * the first device call). The caller guarantees that work enqueued through the context on
 * a previously bound stream is complete or ordered before work on the new one. */
APMM_API int apmm_ctx_set_stream(apmm_ctx* ctx, apmm_stream_t stream);
/* Human-readable message for the last failing call on this thread. */
APMM_API const char* apmm_last_error(void);
APMM_API const char* apmm_status_name(int status);
/* Library build/version string. */
APMM_API const char* apmm_version(void);
/* Number of kernel launches this context has enqueued (launch accounting for bench). */
APMM_API uint64_t apmm_ctx_launch_count(const apmm_ctx* ctx);

/* Pre-size the workspace for calls up to this shape (every route the shape can take), so
 * that no later call grows it -- required before capturing such calls into a CUDA graph.
 * rows_x = feature rows (tokens); n_w is the widest weight width that will be used. */
APMM_API int apmm_ctx_reserve(apmm_ctx* ctx, uint64_t rows_w, uint64_t rows_x, uint64_t k,
                              int n_w);

/* Context options (apmm_ctx_set_option / apmm_ctx_get_option). */
enum {
  /* Kernel route for matmul calls. Routes are schedules only: every route returns the
   * same bits (like TileConfig). AUTO picks by shape; the others
   * force one route and make a call the route cannot serve fail with
   * APMM_E_INVALID_ARGUMENT. Used by the parity tests to pin every kernel. */
  APMM_OPT_ROUTE = 1,
  /* 1 (default): PDL early read of the weight planes (see Conventions); 0: every operand
   * is read after the previous kernel in the stream completed. */
  APMM_OPT_EARLY_WEIGHT_READ = 2,
  /* 0 (default): feature planes are read only after the previous kernel in the stream has
   * completed. 1: they are read early too (more overlap of consecutive calls) -- only for
   * callers whose features are never produced by an early-triggering kernel launched
   * immediately before the call (e.g. several projections of one resident activation). */
  APMM_OPT_EARLY_FEATURE_READ = 3
};
enum {
  APMM_ROUTE_AUTO = 0,         /* by shape */
  APMM_ROUTE_SKINNY = 1,       /* K5: weight planes streamed into mma.sync (rows_x <= 63) */
  APMM_ROUTE_MID_SPLITK = 2,   /* K3f split-K: on-chip weight expansion, K over CTA pairs */
  APMM_ROUTE_PAIR = 3,         /* K1 + K3: tcgen05 cta_group::2 256x256 tiles */
  APMM_ROUTE_PAIR_WPLANES = 4, /* K1(X) + K3f: pair tiles, weights expanded on chip */
  APMM_ROUTE_PAIR_SPLITK = 5,  /* K1 + K3 with K split over the pairs */
  APMM_ROUTE_SINGLE_SM = 6,    /* K1 + K3': 1-SM 128x256 tiles */
  APMM_ROUTE_TENSOR_CORE = 7,  /* AUTO without K5 (tcgen05 routes only) */
  APMM_ROUTE_STREAM_TC = 8     /* K6: weight planes streamed into TMEM (A operand), rows_x <= 128, rows_x % 4 == 0 */
};
APMM_API int apmm_ctx_set_option(apmm_ctx* ctx, int option, int value);
APMM_API int apmm_ctx_get_option(const apmm_ctx* ctx, int option, int* value);

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

/* dot_1bit_xor (kernel.hpp:61-62, kernel.cpp:115-123): k - 2 popc(a ^ b) over exactly
 * ceil(k/32) words of each operand, into *out (device int64). k == 0 -> OutOfRange;
 * a_words or b_words != ceil(k/32) -> LengthMismatch (checked on the host, before any
 * device work). Padding bits are not masked, as in the reference. */
APMM_API int apmm_cu_dot_1bit_xor(apmm_ctx* ctx, const uint32_t* a, uint64_t a_words,
                                  const uint32_t* b, uint64_t b_words, uint64_t k, int64_t* out,
                                  apmm_stream_t stream);

/* Next-layer requantization fused behind the GEMM: matmul_ap with
 * the dequant epilogue (tools/apmm.cpp:329-340) whose f32 output, read as the next layer's
 * activation X' = dequant(Y)^T [rows_x tokens x rows_w features], is quantized
 * (bipolar.cpp:72-100, fp64, per-tensor or per-token) and packed (bitplane.cpp:48-66) into
 * X' planes [n_next][rows_x][ceil(rows_w/32)] + scales (1 or rows_x doubles). Bit-identical
 * to apmm_cu_quantize_pack(transpose((double)apmm_cu_matmul_ap_dequant(...))). The GEMM
 * epilogue also forms the per-token (or global) absmax of its tile, so the requantizer
 * reads the f32 output once. `yf` (device, rows_w x rows_x f32) receives the dequantized
 * output as well (it is the requantizer's input).
 * `absmax` (device, rows_x doubles for per-token, 1 for per-tensor) may be NULL. When given
 * the call stops after the GEMM: absmax receives the local maxima (for a cross-GPU
 * max all-reduce of N-sharded layers) and apmm_cu_requant_pack finishes the job. */
APMM_API int apmm_cu_matmul_ap_requant(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                                       int n_w, const double* w_scales, int w_granularity,
                                       const uint32_t* x_planes, uint64_t rows_x, int n_x,
                                       const double* x_scales, int x_granularity, uint64_t k,
                                       int n_next, int next_granularity, float* yf,
                                       uint32_t* next_planes, double* next_scales,
                                       double* absmax, apmm_stream_t stream);
/* Second half of the split form: quantize + pack yf^T with the given (globally reduced)
 * absmax (rows_x doubles per-token, 1 per-tensor) -> next_planes [n_next][rows_x]
 * [ceil(rows_w/32)] / next_scales. An N-shard's block of the next-layer activation is a
 * column block of whole words when its row count is a multiple of 32, so the blocks of all
 * ranks all-gather into the full activation with one word-block re-layout. Non-finite
 * input -> APMM_E_NON_FINITE after a stream synchronisation, as apmm_cu_quantize_pack. */
APMM_API int apmm_cu_requant_pack(apmm_ctx* ctx, const float* yf, uint64_t rows_w,
                                  uint64_t rows_x, const double* absmax, int n_next,
                                  int next_granularity, uint32_t* next_planes,
                                  double* next_scales, apmm_stream_t stream);

/* ---- APMM v1 tensor files (tensor_file.hpp:12-64) --------------------------------- */
typedef struct apmm_tensor_info {
  int kind;           /* 0 float32 matrix, 1 quantized bipolar (TensorKind) */
  int bit_width;      /* n (0 for float) */
  int granularity;    /* APMM_PER_TENSOR / APMM_PER_ROW, -1 for float */
  uint64_t rows, cols;
  uint64_t scale_count;      /* 1 or rows (quantized), 0 (float) */
  uint64_t payload_offset;   /* byte offset of the f32 values / packed words */
  uint64_t payload_words;    /* rows*cols (float) or n*rows*ceil(cols/32) (quantized) */
} apmm_tensor_info;
/* parse_tensor (tensor_file.cpp:159-229): validates the header, the scales (finite,
 * positive) and the exact payload length -> APMM_E_PARSE with the reference's messages;
 * a quantized payload's padding bits are checked like to_packed -> PackedBitPlanes
 * (bitplane.cpp:22-32, APMM_E_OUT_OF_RANGE). Host only, no device work. */
APMM_API int apmm_tensor_parse(const uint8_t* bytes, uint64_t n_bytes, apmm_tensor_info* info);
/* Parse + upload straight into device buffers (to_packed, tensor_file.cpp:124-130, without
 * the host copy): quantized kind -> planes (n*rows*ceil(cols/32) u32, the PackedBitPlanes
 * layout verbatim) and scales (scale_count doubles); float kind -> values (rows*cols
 * doubles, widened from f32 on the device like to_real, tensor_file.cpp:115-120).
 * Unused pointers may be NULL. Stream-ordered; `bytes` must stay valid until the stream
 * reaches the copy (pinned memory makes it asynchronous). */
APMM_API int apmm_cu_tensor_upload(apmm_ctx* ctx, const uint8_t* bytes, uint64_t n_bytes,
                                   uint32_t* planes, double* scales, double* values,
                                   apmm_stream_t stream);
/* read_tensor_file (tensor_file.cpp:231-) + apmm_cu_tensor_upload, synchronous. A file
 * that cannot be read -> APMM_E_IO. `info` may be NULL. */
APMM_API int apmm_tensor_file_load(apmm_ctx* ctx, const char* path, apmm_tensor_info* info,
                                   uint32_t* planes, double* scales, double* values);
/* serialize_tensor (tensor_file.cpp:135-157) of a quantized tensor from host buffers:
 * writes the exact byte image into out (capacity out_cap) and its length into *out_len.
 * With out == NULL only *out_len is set. */
APMM_API int apmm_tensor_serialize_quantized(uint64_t rows, uint64_t cols, int n,
                                             int granularity, const double* scales,
                                             const uint32_t* planes, uint8_t* out,
                                             uint64_t out_cap, uint64_t* out_len);

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

/* dot_1bit_xor (kernel.cpp:115-123) with host buffers. */
APMM_API int apmm_dot_1bit_xor(apmm_ctx* ctx, const uint32_t* a, uint64_t a_words,
                               const uint32_t* b, uint64_t b_words, uint64_t k, int64_t* out);

/* matmul_plane_pair (kernel.cpp:125-144) with host buffers; validates padding. */
APMM_API int apmm_matmul_plane_pair(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                                    int n_w, int weight_plane, const uint32_t* x_planes,
                                    uint64_t rows_x, int n_x, int feature_plane, uint64_t k,
                                    int32_t* y);

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
