// apmm_cuda.cu -- the C ABI (include/apmm_cuda.h): validation with the reference's error
// semantics, workspace management, and dispatch onto the sm_100a kernels.
//
// Validation order follows the reference so the same inputs fail with the same error
// class: BitWidth (bipolar.hpp:17-19) -> positive dimensions (bitplane.cpp:14-16) ->
// buffer contents (bitplane.cpp:22-32) -> K agreement / overflow_bound (kernel.cpp:189-199).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/apmm_cuda.h"
#include "internal.h"

using namespace apmm_b200;

struct apmm_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* ws = nullptr;  // matmul workspace (u8 codes + rowsums + scratch)
  size_t ws_bytes = 0;
  void* io = nullptr;  // device staging for the synchronous host entry points
  size_t io_bytes = 0;
  uint64_t launches = 0;
  // measurement: event pairs around launches of kernel class 0 (GEMM) / 1 (expand)
  bool timing = false;
  bool force_single_sm = false;
  int ws_half = 0;  // which half of the ping-pong workspace the next matmul uses
  void* sk_ws = nullptr;  // K5 split-K accumulators (zero between calls)
  size_t sk_ws_bytes = 0;
  void* sk_scratch = nullptr;  // K5 feature fragments (ping-pong halves) + weight repack
  size_t sk_scratch_bytes = 0;
  bool force_tc = false;  // APMM_FORCE_TC=1: never use K5 (testing)
  bool dbg_waits = false;  // APMM_DEBUG_WAITS=1: MMA-issuer wait-cycle counters (dev only)
  void* dbg = nullptr;  // APMM_DEBUG_WAITS counters (dev only)
  int* flags = nullptr;  // recover's device error flags (2 ints)
  void* qx = nullptr;  // fused quantize: feature planes (skinny) / absmax + flag scratch
  size_t qx_bytes = 0;
  // host entry points' transfer pipeline: H2D / D2H copy streams and their events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t pipe_ev[16] = {};
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[2];
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> spare;
};

namespace {

constexpr uint64_t kPipeBlocks = 8;  // host_matmul row blocks in flight (events: 2 per block)

thread_local std::string g_last_error;

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(APMM_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CU(expr)                                        \
  do {                                                  \
    cudaError_t e_ = (expr);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)

constexpr size_t kAlign = 1024;
size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

int check_width(int n) {
  if (n < 1 || n > 8) return fail(APMM_E_OUT_OF_RANGE, "bit width must be in [1, 8], got %d", n);
  return APMM_OK;
}

int check_dims(uint64_t rows, uint64_t cols, const char* what) {
  if (rows == 0 || cols == 0) {
    return fail(APMM_E_DIMENSION_MISMATCH, "%s dimensions must be positive", what);
  }
  if (rows >= (1ull << 31) || cols >= (1ull << 31)) {
    return fail(APMM_E_INVALID_ARGUMENT, "%s dimensions exceed 2^31-1", what);
  }
  return APMM_OK;
}

int64_t bound_of(int n_w, int n_x, uint64_t k) {
  return static_cast<int64_t>(k) * ((1 << n_w) - 1) * ((1 << n_x) - 1);
}

int check_matmul(int n_w, int n_x, uint64_t rows_w, uint64_t rows_x, uint64_t k) {
  int st;
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  if ((st = check_dims(rows_w, k, "weights")) || (st = check_dims(rows_x, k, "features"))) {
    return st;
  }
  const int64_t b = bound_of(n_w, n_x, k);
  if (b > INT32_MAX) {
    return fail(APMM_E_OVERFLOW_BOUND,
                "output bound %lld exceeds 32-bit range; K=%llu n_w=%d n_x=%d",
                static_cast<long long>(b), static_cast<unsigned long long>(k), n_w, n_x);
  }
  return APMM_OK;
}

int ensure(void** buf, size_t* have, size_t need, int device) {
  if (need <= *have) return APMM_OK;
  CU(cudaSetDevice(device));
  if (*buf) {
    CU(cudaDeviceSynchronize());  // growth only: previous users of the buffer must finish
    CU(cudaFree(*buf));
    *buf = nullptr;
    *have = 0;
  }
  const size_t sz = need + need / 4;
  CU(cudaMalloc(buf, sz));
  *have = sz;
  return APMM_OK;
}

// Workspace carve-up for one matmul.
struct MatmulWs {
  uint8_t* codes_w;
  uint8_t* codes_x;
  int32_t* rowsum_w;
  int32_t* rowsum_x;
  uint64_t kpad;
};

// Two halves (ping-pong): consecutive calls alternate, so the next call's expand can run
// while this call's GEMM still reads its half (PDL overlap, see prep.cu / gemm_pair.cu).
size_t matmul_half_bytes(uint64_t rows_w, uint64_t rows_x, uint64_t k) {
  const uint64_t kpad = round_up(k, kKAlign);
  return align_up(rows_w * kpad) + align_up(rows_x * kpad) + align_up(rows_w * 4) +
         align_up(round_up(rows_x, kRowsumPad) * 4);
}

size_t matmul_ws_bytes(uint64_t rows_w, uint64_t rows_x, uint64_t k) {
  return 2 * matmul_half_bytes(rows_w, rows_x, k);
}

MatmulWs carve(void* ws, uint64_t rows_w, uint64_t rows_x, uint64_t k, int half) {
  MatmulWs m;
  m.kpad = round_up(k, kKAlign);
  uint8_t* p = static_cast<uint8_t*>(ws) + (half ? matmul_half_bytes(rows_w, rows_x, k) : 0);
  m.codes_w = p;
  p += align_up(rows_w * m.kpad);
  m.codes_x = p;
  p += align_up(rows_x * m.kpad);
  m.rowsum_w = reinterpret_cast<int32_t*>(p);
  p += align_up(rows_w * 4);
  m.rowsum_x = reinterpret_cast<int32_t*>(p);
  return m;
}

// Event bracket around one launch when timing is enabled.
struct TimedLaunch {
  apmm_ctx* ctx;
  int kind;
  cudaStream_t s;
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  unsigned flags = cudaEventRecordDefault;
  bool record;
  TimedLaunch(apmm_ctx* c, int k, cudaStream_t st, bool rec = true)
      : ctx(c), kind(k), s(st), record(rec) {
    if (!ctx->timing) return;
    if (!ctx->spare.empty()) {
      ev = ctx->spare.back();
      ctx->spare.pop_back();
    } else {
      cudaEventCreate(&ev.first);
      cudaEventCreate(&ev.second);
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    // inside a stream capture the records must be external event-record nodes, so the
    // events are really recorded (and timed) when the graph is replayed
    flags = cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
    if (record) cudaEventRecordWithFlags(ev.first, s, flags);
  }
  ~TimedLaunch() {
    if (!ctx->timing) return;
    if (record) cudaEventRecordWithFlags(ev.second, s, flags);
    ctx->pending[kind].push_back(ev);
  }
};

// x_ready: the feature operand is already in this call's workspace half as u8 codes +
// rowsum (written by the fused quantize, K2 -> K3); then K1 expands W only and x is unused.
int run_matmul(apmm_ctx* ctx, const uint32_t* w, uint64_t rows_w, int n_w, const double* s_w,
               int gran_w, const uint32_t* x, uint64_t rows_x, int n_x, const double* s_x,
               int gran_x, uint64_t k, int32_t* y, float* yf, cudaStream_t stream,
               bool x_ready = false) {
  CU(cudaSetDevice(ctx->device));
  // Route. CTA-pair 256x256 tiles (K3) when they fill the machine. Otherwise mid-size calls
  // (M_tok <= 256) take the split-K K3f: the weight planes are expanded on chip (each W row
  // once: a single N tile), rowsum(U_w) formed by the transform warps, K split across CTA
  // pairs, int32 partials TMA reduce-added into a Y zeroed by K1 (4096x128x4096 W2A4: 14.0
  // us vs 18.3 us for K1 + the 1-SM GEMM; profiles/r01b_mid_size_v2.txt). Feature counts up
  // to kSkinnyPreferRows stay on K5 (faster there: 4096x40x4096 8.6 vs 12.6 us,
  // profiles/r01b_skinny_mid_boundary.txt), and K5 takes up to 63 rows when the split-K
  // path cannot (int32 output with a TMA-storable Y only). APMM_MID=0/1 forces the split-K
  // path off/on, APMM_SKINNY_MAX moves the K5 boundary (testing).
  const uint64_t pair_tiles = ((rows_w + 255) / 256) * ((rows_x + kPairN - 1) / kPairN);
  const bool pair = pair_tiles >= static_cast<uint64_t>(ctx->num_sms / 2) && !ctx->force_single_sm;
  const char* mid_env = std::getenv("APMM_MID");
  const bool mid = (mid_env ? mid_env[0] == '1' : rows_x <= 256) && !pair &&
                   !ctx->force_single_sm && !yf && rows_x > 0 && rows_x % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(y) % 16 == 0 && gemm_wplanes_addressable(w, k);
  static const uint64_t skinny_prefer = [] {
    const char* e = std::getenv("APMM_SKINNY_MAX");
    return e ? static_cast<uint64_t>(std::atoll(e)) : kSkinnyPreferRows;
  }();
  const bool skinny = rows_x <= kSkinnyMaxRowsX && !ctx->force_tc && !x_ready &&
                      (rows_x <= skinny_prefer || !mid);
  if (skinny) {
    // few feature rows: feature prep + K5, the weight planes streamed once from HBM
    const size_t need = skinny_acc_bytes(rows_w, rows_x);
    if (need > ctx->sk_ws_bytes) {  // split-K accumulators; zero at rest
      if (ctx->sk_ws) {
        CU(cudaDeviceSynchronize());
        CU(cudaFree(ctx->sk_ws));
        ctx->sk_ws = nullptr;
        ctx->sk_ws_bytes = 0;
      }
      const size_t sz = need + need / 4;
      CU(cudaMalloc(&ctx->sk_ws, sz));
      CU(cudaMemset(ctx->sk_ws, 0, sz));
      ctx->sk_ws_bytes = sz;
    }
    int st = ensure(&ctx->sk_scratch, &ctx->sk_scratch_bytes,
                    skinny_scratch_bytes(rows_w, rows_x, k, n_w, w), ctx->device);
    if (st) return st;
    SkinnyArgs s{};
    s.w_planes = w;
    s.x_planes = x;
    s.rows_w = rows_w;
    s.rows_x = rows_x;
    s.k = k;
    s.n_w = n_w;
    s.n_x = n_x;
    s.y = y;
    s.yf = yf;
    s.s_w = s_w;
    s.gran_w = gran_w;
    s.s_x = s_x;
    s.gran_x = gran_x;
    s.num_sms = ctx->num_sms;
    s.acc_ws = ctx->sk_ws;
    s.scratch_ws = ctx->sk_scratch;
    s.ws_half = ctx->ws_half;
    ctx->ws_half ^= 1;
    {
      // kernel timing brackets the streaming kernel alone (not the feature-prep launch)
      TimedLaunch t(ctx, 0, stream, /*record=*/false);
      s.ev_start = t.ev.first;
      s.ev_stop = t.ev.second;
      s.ev_flags = t.flags;
      CU(launch_skinny(s, stream));
    }
    ctx->launches += rows_x <= 1 ? 1 : 2;  // (feature prep +) streaming kernel
    return APMM_OK;
  }
  int st = ensure(&ctx->ws, &ctx->ws_bytes, matmul_ws_bytes(rows_w, rows_x, k), ctx->device);
  if (st) return st;
  const MatmulWs m = carve(ctx->ws, rows_w, rows_x, k, ctx->ws_half);
  ctx->ws_half ^= 1;
  const uint64_t rsx_pad = round_up(rows_x, kRowsumPad);
  const bool fused = pair && gemm_fused_supported(w, k);
  // Opt-in (APMM_PSPLIT=1): the u8-code pair GEMM with K split over the pairs (partials
  // reduce-added into a Y zeroed by K1) for calls with too few pair tiles. Bit-exact, but
  // measured slower than the 1-SM kernel for 256 < M_tok <= 1024 (4096x512x4096: 32.4 vs
  // 20.3 us; profiles/r01b_pair_split_sweep.txt).
  const char* ps_env = std::getenv("APMM_PSPLIT");
  const bool psplit = ps_env != nullptr && ps_env[0] == '1' && !pair && !mid &&
                      !ctx->force_single_sm && !yf && rows_x % 4 == 0 &&
                      reinterpret_cast<uintptr_t>(y) % 16 == 0;
  {
    TimedLaunch t(ctx, 1, stream);
    // mid (split-K K3f): W untouched (the GEMM expands it and forms rowsum(U_w) itself);
    // K1 expands X and zeroes Y, which the split-K units reduce-add into
    CU(launch_expand(w, mid ? 0 : rows_w, n_w, (fused || mid) ? nullptr : m.codes_w, m.rowsum_w,
                     x_ready ? nullptr : x, x_ready ? 0 : rows_x, x_ready ? 0 : rsx_pad, n_x,
                     m.codes_x, m.rowsum_x, k, m.kpad, ctx->num_sms, stream,
                     (mid || psplit) ? static_cast<void*>(y) : nullptr,
                     (mid || psplit) ? rows_w * rows_x * 4 : 0));
  }
  ctx->launches += 1;
  GemmArgs a{};
  a.codes_w = m.codes_w;
  a.codes_x = m.codes_x;
  a.rowsum_w = m.rowsum_w;
  a.rowsum_x = m.rowsum_x;
  a.rows_w = rows_w;
  a.rows_x = rows_x;
  a.kpad = m.kpad;
  a.k_logical = k;
  a.n_w = n_w;
  a.n_x = n_x;
  a.y = y;
  a.yf = yf;
  a.s_w = s_w;
  a.gran_w = gran_w;
  a.s_x = s_x;
  a.gran_x = gran_x;
  a.num_sms = ctx->num_sms;
  if (ctx->dbg_waits) {
    if (!ctx->dbg) {
      CU(cudaMalloc(&ctx->dbg, 128));
      CU(cudaMemset(ctx->dbg, 0, 128));
    }
    a.dbg = static_cast<unsigned long long*>(ctx->dbg);
  }
  int launches = 0;
  {
    TimedLaunch t(ctx, 0, stream);
    if (fused || mid) {
      CU(launch_gemm_pair_wplanes(a, w, stream, &launches, /*split_k=*/mid));
    } else if (pair || psplit) {
      CU(launch_gemm_pair(a, stream, &launches, /*split_k=*/psplit));
    } else {
      CU(launch_gemm_tc(a, stream, &launches));
    }
  }
  ctx->launches += static_cast<uint64_t>(launches);
  return APMM_OK;
}

// Device entry points run on exactly the stream they are given (NULL = the legacy default
// stream, as everywhere in CUDA); only the host entry points use the context's stream.
cudaStream_t pick(apmm_ctx* /*ctx*/, apmm_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Host-side PackedBitPlanes invariants (bitplane.cpp:17-32).
int check_padding(const uint32_t* planes, uint64_t rows, uint64_t cols, int n) {
  const uint32_t tail = static_cast<uint32_t>(cols & 31);
  if (tail == 0) return APMM_OK;
  const uint32_t pad = ~((1u << tail) - 1u);
  const uint64_t wpr = (cols + 31) / 32;
  for (uint64_t pr = 0; pr < uint64_t(n) * rows; ++pr) {
    if (planes[(pr + 1) * wpr - 1] & pad) {
      return fail(APMM_E_OUT_OF_RANGE, "packed buffer has nonzero padding bits");
    }
  }
  return APMM_OK;
}

bool valid_gran(int g) { return g == APMM_PER_TENSOR || g == APMM_PER_ROW; }

}  // namespace

extern "C" {

const char* apmm_last_error(void) { return g_last_error.c_str(); }

const char* apmm_status_name(int s) {
  switch (s) {
    case APMM_OK: return "OK";
    case APMM_E_EVEN_VALUE: return "EvenValue";
    case APMM_E_OUT_OF_RANGE: return "OutOfRange";
    case APMM_E_NON_FINITE: return "NonFinite";
    case APMM_E_LENGTH_MISMATCH: return "LengthMismatch";
    case APMM_E_DIMENSION_MISMATCH: return "DimensionMismatch";
    case APMM_E_INDEX_OUT_OF_BOUNDS: return "IndexOutOfBounds";
    case APMM_E_OVERFLOW: return "Overflow";
    case APMM_E_OVERFLOW_BOUND: return "OverflowBound";
    case APMM_E_INVALID_ARGUMENT: return "InvalidArgument";
    case APMM_E_CUDA: return "CudaError";
    case APMM_E_NO_DEVICE: return "NoDevice";
    case APMM_E_UNSUPPORTED_DEVICE: return "UnsupportedDevice";
    default: return "Unknown";
  }
}

const char* apmm_version(void) {
  return "apmm_b200 0.1 (sm_100a; tcgen05 kind::i8 u8-code GEMM, rank-1 recovery epilogue)";
}

int apmm_ctx_create(apmm_ctx** out, int device) {
  if (!out) return fail(APMM_E_INVALID_ARGUMENT, "null context pointer");
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(APMM_E_NO_DEVICE, "no CUDA device visible");
  }
  if (device < 0 || device >= count) return fail(APMM_E_NO_DEVICE, "device %d out of range", device);
  cudaDeviceProp prop;
  CU(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0) {
    return fail(APMM_E_UNSUPPORTED_DEVICE, "device %d is sm_%d%d; this library is built for sm_100a",
                device, prop.major, prop.minor);
  }
  CU(cudaSetDevice(device));
  auto* ctx = new apmm_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  if (const char* f = std::getenv("APMM_FORCE_1SM")) ctx->force_single_sm = f[0] == '1';
  if (const char* f = std::getenv("APMM_DEBUG_WAITS")) ctx->dbg_waits = f[0] == '1';
  if (const char* f = std::getenv("APMM_FORCE_TC")) ctx->force_tc = f[0] == '1';
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_fail(e, "cudaStreamCreate");
  }
  ctx->own_stream = true;
  *out = ctx;
  return APMM_OK;
}

int apmm_ctx_destroy(apmm_ctx* ctx) {
  if (!ctx) return APMM_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  if (ctx->dbg) {
    unsigned long long h[16] = {};
    cudaMemcpy(h, ctx->dbg, sizeof(h), cudaMemcpyDeviceToHost);
    std::fprintf(stderr,
                 "[apmm debug] MMA issuer: %.1f%% of cycles waiting on operands (full), %.1f%% on "
                 "epilogue (tmem_empty), over %llu issuer runs\n",
                 h[2] ? 100.0 * h[0] / h[2] : 0.0, h[2] ? 100.0 * h[1] / h[2] : 0.0, h[3]);
    if (h[8]) {
      std::fprintf(stderr,
                   "[apmm debug] fused transform warps: %.1f%% waiting for free operand slots, "
                   "%.1f%% storing + next block's planes -> codes (of which %.1f%% waiting for "
                   "raw planes), %.1f%% fence + arrive; "
                   "%.0f cycles per warp run over %llu runs\n",
                   h[7] ? 100.0 * h[4] / h[7] : 0.0, h[7] ? 100.0 * h[5] / h[7] : 0.0,
                   h[7] ? 100.0 * h[9] / h[7] : 0.0, h[7] ? 100.0 * h[6] / h[7] : 0.0, double(h[7]) / h[8], h[8]);
    }
    cudaFree(ctx->dbg);
  }
  if (ctx->flags) cudaFree(ctx->flags);
  if (ctx->qx) cudaFree(ctx->qx);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->sk_ws) cudaFree(ctx->sk_ws);
  if (ctx->sk_scratch) cudaFree(ctx->sk_scratch);
  if (ctx->io) cudaFree(ctx->io);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->s_in) cudaStreamDestroy(ctx->s_in);
  if (ctx->s_out) cudaStreamDestroy(ctx->s_out);
  for (auto& e : ctx->pipe_ev) {
    if (e) cudaEventDestroy(e);
  }
  for (auto* v : {&ctx->pending[0], &ctx->pending[1], &ctx->spare}) {
    for (auto& ev : *v) {
      cudaEventDestroy(ev.first);
      cudaEventDestroy(ev.second);
    }
  }
  delete ctx;
  return APMM_OK;
}

int apmm_ctx_set_stream(apmm_ctx* ctx, apmm_stream_t stream) {
  if (!ctx) return fail(APMM_E_INVALID_ARGUMENT, "null context");
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  ctx->stream = reinterpret_cast<cudaStream_t>(stream);
  ctx->own_stream = false;
  return APMM_OK;
}

uint64_t apmm_ctx_launch_count(const apmm_ctx* ctx) { return ctx ? ctx->launches : 0; }

int apmm_ctx_enable_timing(apmm_ctx* ctx, int enable) {
  if (!ctx) return fail(APMM_E_INVALID_ARGUMENT, "null context");
  ctx->timing = enable != 0;
  return APMM_OK;
}

int apmm_ctx_kernel_time(apmm_ctx* ctx, int kernel, double* total_ms, uint64_t* launches) {
  if (!ctx || !total_ms || !launches || kernel < 0 || kernel > 1) {
    return fail(APMM_E_INVALID_ARGUMENT, "bad argument");
  }
  CU(cudaSetDevice(ctx->device));
  double sum = 0.0;
  for (auto& ev : ctx->pending[kernel]) {
    CU(cudaEventSynchronize(ev.second));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, ev.first, ev.second));
    sum += ms;
    ctx->spare.push_back(ev);
  }
  *launches = ctx->pending[kernel].size();
  *total_ms = sum;
  ctx->pending[kernel].clear();
  return APMM_OK;
}

int apmm_overflow_bound(int n_w, int n_x, uint64_t k, int64_t* bound) {
  int st;
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  if (!bound) return fail(APMM_E_INVALID_ARGUMENT, "null output");
  *bound = bound_of(n_w, n_x, k);
  return APMM_OK;
}

uint64_t apmm_packed_words(int n, uint64_t rows, uint64_t cols) {
  return static_cast<uint64_t>(n) * rows * ((cols + 31) / 32);
}

// ---- device entry points ----------------------------------------------------------------
int apmm_cu_pack(apmm_ctx* ctx, const uint8_t* codes, uint64_t rows, uint64_t cols, int n,
                 uint32_t* planes, apmm_stream_t stream) {
  int st;
  if (!ctx || !codes || !planes) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "CodeMatrix"))) return st;
  CU(cudaSetDevice(ctx->device));
  CU(launch_pack(codes, rows, cols, n, planes, pick(ctx, stream)));
  ctx->launches += 1;
  return APMM_OK;
}

int apmm_cu_unpack(apmm_ctx* ctx, const uint32_t* planes, uint64_t rows, uint64_t cols, int n,
                   uint8_t* codes, apmm_stream_t stream) {
  int st;
  if (!ctx || !codes || !planes) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "PackedBitPlanes"))) return st;
  CU(cudaSetDevice(ctx->device));
  CU(launch_unpack(planes, rows, cols, n, codes, pick(ctx, stream)));
  ctx->launches += 1;
  return APMM_OK;
}

int apmm_cu_quantize_pack(apmm_ctx* ctx, const double* values, uint64_t rows, uint64_t cols,
                          int n, int granularity, uint32_t* planes, double* scales,
                          uint8_t* codes, apmm_stream_t stream) {
  int st;
  if (!ctx || !values || !planes || !scales) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if (!valid_gran(granularity)) return fail(APMM_E_INVALID_ARGUMENT, "bad granularity");
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "RealMatrix"))) return st;
  // scratch: amax bits + flag live past the matmul region of the workspace
  if ((st = ensure(&ctx->ws, &ctx->ws_bytes, 64, ctx->device))) return st;
  CU(cudaSetDevice(ctx->device));
  auto* amax = static_cast<unsigned long long*>(ctx->ws);
  int* flag = reinterpret_cast<int*>(static_cast<uint8_t*>(ctx->ws) + 16);
  const cudaStream_t s = pick(ctx, stream);
  CU(launch_quantize_pack(values, rows, cols, n, granularity, planes, scales, codes, amax, flag, s));
  ctx->launches += granularity == APMM_PER_ROW ? 1 : 2;
  int h_flag = 0;
  CU(cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (h_flag) return fail(APMM_E_NON_FINITE, "input contains NaN or infinity");
  return APMM_OK;
}

int apmm_cu_matmul_ap(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                      const uint32_t* x_planes, uint64_t rows_x, int n_x, uint64_t k,
                      int32_t* y, apmm_stream_t stream) {
  if (!ctx || !w_planes || !x_planes || !y) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  int st = check_matmul(n_w, n_x, rows_w, rows_x, k);
  if (st) return st;
  return run_matmul(ctx, w_planes, rows_w, n_w, nullptr, 0, x_planes, rows_x, n_x, nullptr, 0, k,
                    y, nullptr, pick(ctx, stream));
}

int apmm_cu_matmul_ap_dequant(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                              int n_w, const double* w_scales, int w_granularity,
                              const uint32_t* x_planes, uint64_t rows_x, int n_x,
                              const double* x_scales, int x_granularity, uint64_t k,
                              float* out, apmm_stream_t stream) {
  if (!ctx || !w_planes || !x_planes || !out || !w_scales || !x_scales) {
    return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  }
  if (!valid_gran(w_granularity) || !valid_gran(x_granularity)) {
    return fail(APMM_E_INVALID_ARGUMENT, "bad granularity");
  }
  int st = check_matmul(n_w, n_x, rows_w, rows_x, k);
  if (st) return st;
  return run_matmul(ctx, w_planes, rows_w, n_w, w_scales, w_granularity, x_planes, rows_x, n_x,
                    x_scales, x_granularity, k, nullptr, out, pick(ctx, stream));
}

int apmm_cu_matmul_plane_pair(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                              int weight_plane, const uint32_t* x_planes, uint64_t rows_x,
                              int n_x, int feature_plane, uint64_t k, int32_t* y,
                              apmm_stream_t stream) {
  int st;
  if (!ctx || !w_planes || !x_planes || !y) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  if (weight_plane < 0 || weight_plane >= n_w || feature_plane < 0 || feature_plane >= n_x) {
    return fail(APMM_E_INDEX_OUT_OF_BOUNDS, "plane pair (%d, %d) out of range", weight_plane,
                feature_plane);
  }
  // one plane of a packed buffer is itself a 1-bit packed buffer; a 1-bit x 1-bit matmul_ap
  // is exactly the XOR dot  K - 2 popc(a ^ b)  of kernel.cpp:115-144 (v = 2u - 1 = +-1)
  if ((st = check_matmul(1, 1, rows_w, rows_x, k))) return st;
  const uint64_t wpr = (k + 31) / 32;
  return run_matmul(ctx, w_planes + uint64_t(weight_plane) * rows_w * wpr, rows_w, 1, nullptr, 0,
                    x_planes + uint64_t(feature_plane) * rows_x * wpr, rows_x, 1, nullptr, 0, k,
                    y, nullptr, pick(ctx, stream));
}

int apmm_cu_compute_plane_products(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                                   int n_w, const uint32_t* x_planes, uint64_t rows_x, int n_x,
                                   uint64_t k, int32_t* stack, apmm_stream_t stream) {
  if (!ctx || !stack) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  int st;
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  for (int i = 0; i < n_w; ++i) {
    for (int j = 0; j < n_x; ++j) {
      st = apmm_cu_matmul_plane_pair(ctx, w_planes, rows_w, n_w, i, x_planes, rows_x, n_x, j, k,
                                     stack + uint64_t(i * n_x + j) * rows_w * rows_x, stream);
      if (st) return st;
    }
  }
  return APMM_OK;
}

int apmm_cu_recover(apmm_ctx* ctx, const int32_t* stack, int n_w, int n_x, uint64_t k,
                    uint64_t rows, uint64_t cols, int32_t* y, apmm_stream_t stream) {
  int st;
  if (!ctx || !stack || !y) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  CU(cudaSetDevice(ctx->device));
  if (!ctx->flags) CU(cudaMalloc(&ctx->flags, 2 * sizeof(int)));
  const cudaStream_t s = pick(ctx, stream);
  CU(cudaMemsetAsync(ctx->flags, 0, 2 * sizeof(int), s));
  CU(launch_recover(stack, n_w, n_x, rows * cols, k, y, ctx->flags, s));
  ctx->launches += 1;
  int h[2] = {0, 0};
  CU(cudaMemcpyAsync(h, ctx->flags, sizeof(h), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (h[0]) return fail(APMM_E_OUT_OF_RANGE, "plane product entry outside [-K, K]");
  if (h[1]) return fail(APMM_E_OVERFLOW, "recovered value exceeds 32-bit range");
  return APMM_OK;
}

int apmm_cu_quantize_matmul_ap_dequant(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                                       int n_w, const double* w_scales, int w_granularity,
                                       const double* x_values, uint64_t rows_x, uint64_t k,
                                       int n_x, int x_granularity, double* x_scales, float* out,
                                       apmm_stream_t stream) {
  int st;
  if (!ctx || !w_planes || !w_scales || !x_values || !x_scales || !out) {
    return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  }
  if (!valid_gran(w_granularity) || !valid_gran(x_granularity)) {
    return fail(APMM_E_INVALID_ARGUMENT, "bad granularity");
  }
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  if ((st = check_dims(rows_x, k, "RealMatrix")) || (st = check_dims(rows_w, k, "weights"))) return st;
  CU(cudaSetDevice(ctx->device));
  const cudaStream_t s = pick(ctx, stream);
  if (rows_x <= kSkinnyMaxRowsX && !ctx->force_tc) {
    // few feature rows: the skinny kernel consumes planes -> quantize_pack into a scratch
    // plane buffer, then the ordinary device matmul (both stream-ordered)
    const size_t words = apmm_packed_words(n_x, rows_x, k);
    if ((st = ensure(&ctx->qx, &ctx->qx_bytes, words * 4 + 64, ctx->device))) return st;
    uint32_t* xp = static_cast<uint32_t*>(ctx->qx);
    if ((st = apmm_cu_quantize_pack(ctx, x_values, rows_x, k, n_x, x_granularity, xp, x_scales,
                                    nullptr, stream))) {
      return st;
    }
    if ((st = check_matmul(n_w, n_x, rows_w, rows_x, k))) return st;
    return run_matmul(ctx, w_planes, rows_w, n_w, w_scales, w_granularity, xp, rows_x, n_x,
                      x_scales, x_granularity, k, nullptr, out, s);
  }
  // K2 -> K3: quantize straight into this call's workspace half (u8 codes in K1's layout +
  // rowsum(U_x)); K1 then expands W only. The feature planes never exist.
  if ((st = ensure(&ctx->ws, &ctx->ws_bytes, matmul_ws_bytes(rows_w, rows_x, k), ctx->device))) return st;
  if ((st = ensure(&ctx->qx, &ctx->qx_bytes, 64, ctx->device))) return st;
  const MatmulWs m = carve(ctx->ws, rows_w, rows_x, k, ctx->ws_half);
  auto* amax = static_cast<unsigned long long*>(ctx->qx);
  int* flag = reinterpret_cast<int*>(static_cast<uint8_t*>(ctx->qx) + 16);
  CU(launch_quantize_pack(x_values, rows_x, k, n_x, x_granularity, nullptr, x_scales, nullptr,
                          amax, flag, s, m.codes_x, m.rowsum_x, m.kpad, round_up(rows_x, kRowsumPad)));
  ctx->launches += x_granularity == APMM_PER_ROW ? 1 : 2;
  int h_flag = 0;  // quantize errors come first, as in the reference flow (apmm.cpp:275-327)
  CU(cudaMemcpyAsync(&h_flag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (h_flag) return fail(APMM_E_NON_FINITE, "input contains NaN or infinity");
  if ((st = check_matmul(n_w, n_x, rows_w, rows_x, k))) return st;
  return run_matmul(ctx, w_planes, rows_w, n_w, w_scales, w_granularity, nullptr, rows_x, n_x,
                    x_scales, x_granularity, k, nullptr, out, s, /*x_ready=*/true);
}

// ---- host entry points ------------------------------------------------------------------
int apmm_decompose_and_pack(apmm_ctx* ctx, const uint8_t* codes, uint64_t rows, uint64_t cols,
                            int n, uint32_t* planes) {
  int st;
  if (!ctx || !codes || !planes) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "CodeMatrix"))) return st;
  const uint32_t limit = 1u << n;
  for (uint64_t e = 0; e < rows * cols; ++e) {  // CodeMatrix ctor (bipolar.cpp:33-36)
    if (codes[e] >= limit) return fail(APMM_E_OUT_OF_RANGE, "code has bits above position n-1");
  }
  const size_t in_b = align_up(rows * cols), out_b = apmm_packed_words(n, rows, cols) * 4;
  if ((st = ensure(&ctx->io, &ctx->io_bytes, in_b + out_b, ctx->device))) return st;
  uint8_t* d_codes = static_cast<uint8_t*>(ctx->io);
  uint32_t* d_planes = reinterpret_cast<uint32_t*>(d_codes + in_b);
  CU(cudaMemcpyAsync(d_codes, codes, rows * cols, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = apmm_cu_pack(ctx, d_codes, rows, cols, n, d_planes, reinterpret_cast<apmm_stream_t>(ctx->stream)))) return st;
  CU(cudaMemcpyAsync(planes, d_planes, out_b, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return APMM_OK;
}

int apmm_unpack(apmm_ctx* ctx, const uint32_t* planes, uint64_t rows, uint64_t cols, int n,
                uint8_t* codes) {
  int st;
  if (!ctx || !codes || !planes) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "PackedBitPlanes"))) return st;
  if ((st = check_padding(planes, rows, cols, n))) return st;
  const size_t in_b = align_up(apmm_packed_words(n, rows, cols) * 4), out_b = rows * cols;
  if ((st = ensure(&ctx->io, &ctx->io_bytes, in_b + out_b, ctx->device))) return st;
  uint32_t* d_planes = static_cast<uint32_t*>(ctx->io);
  uint8_t* d_codes = static_cast<uint8_t*>(ctx->io) + in_b;
  CU(cudaMemcpyAsync(d_planes, planes, apmm_packed_words(n, rows, cols) * 4,
                     cudaMemcpyHostToDevice, ctx->stream));
  if ((st = apmm_cu_unpack(ctx, d_planes, rows, cols, n, d_codes, reinterpret_cast<apmm_stream_t>(ctx->stream)))) return st;
  CU(cudaMemcpyAsync(codes, d_codes, out_b, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return APMM_OK;
}

int apmm_quantize_pack(apmm_ctx* ctx, const double* values, uint64_t rows, uint64_t cols, int n,
                       int granularity, uint8_t* codes, uint32_t* planes, double* scales) {
  int st;
  if (!ctx || !values || !planes || !scales) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if (!valid_gran(granularity)) return fail(APMM_E_INVALID_ARGUMENT, "bad granularity");
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "RealMatrix"))) return st;
  const uint64_t n_scales = granularity == APMM_PER_ROW ? rows : 1;
  const size_t x_b = align_up(rows * cols * 8), p_b = align_up(apmm_packed_words(n, rows, cols) * 4);
  const size_t s_b = align_up(n_scales * 8), c_b = align_up(rows * cols);
  if ((st = ensure(&ctx->io, &ctx->io_bytes, x_b + p_b + s_b + c_b, ctx->device))) return st;
  uint8_t* base = static_cast<uint8_t*>(ctx->io);
  double* d_x = reinterpret_cast<double*>(base);
  uint32_t* d_p = reinterpret_cast<uint32_t*>(base + x_b);
  double* d_s = reinterpret_cast<double*>(base + x_b + p_b);
  uint8_t* d_c = codes ? base + x_b + p_b + s_b : nullptr;
  CU(cudaMemcpyAsync(d_x, values, rows * cols * 8, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = apmm_cu_quantize_pack(ctx, d_x, rows, cols, n, granularity, d_p, d_s, d_c,
                                   reinterpret_cast<apmm_stream_t>(ctx->stream)))) {
    return st;
  }
  CU(cudaMemcpyAsync(planes, d_p, apmm_packed_words(n, rows, cols) * 4, cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaMemcpyAsync(scales, d_s, n_scales * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (codes) CU(cudaMemcpyAsync(codes, d_c, rows * cols, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return APMM_OK;
}

// Synchronous host entry point. Large calls are pipelined over row blocks of W (= row
// blocks of Y): block b's weight planes go up on a copy stream while block b-1 computes on
// the context stream and block b-2's results come down on a second copy stream, so the
// PCIe transfers in both directions overlap each other and the GEMMs. Small calls run as
// one block.
static int host_matmul(apmm_ctx* ctx, const uint32_t* w, uint64_t rows_w, int n_w,
                       const double* s_w, int gran_w, const uint32_t* x, uint64_t rows_x,
                       int n_x, const double* s_x, int gran_x, uint64_t k, int32_t* y,
                       float* yf) {
  int st;
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  if ((st = check_dims(rows_w, k, "weights")) || (st = check_dims(rows_x, k, "features"))) {
    return st;
  }
  if ((st = check_padding(w, rows_w, k, n_w)) || (st = check_padding(x, rows_x, k, n_x))) {
    return st;
  }
  if ((st = check_matmul(n_w, n_x, rows_w, rows_x, k))) return st;
  const uint64_t wpr = (k + 31) / 32;
  const size_t w_words = apmm_packed_words(n_w, rows_w, k), x_words = apmm_packed_words(n_x, rows_x, k);
  const size_t w_b = align_up(w_words * 4), x_b = align_up(x_words * 4);
  const size_t y_b = align_up(rows_w * rows_x * 4);
  const size_t sw_n = gran_w == APMM_PER_ROW ? rows_w : 1, sx_n = gran_x == APMM_PER_ROW ? rows_x : 1;
  const size_t sw_b = yf ? align_up(sw_n * 8) : 0, sx_b = yf ? align_up(sx_n * 8) : 0;
  if ((st = ensure(&ctx->io, &ctx->io_bytes, w_b + x_b + y_b + sw_b + sx_b, ctx->device))) return st;
  CU(cudaSetDevice(ctx->device));
  if (!ctx->s_in) {
    CU(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
    for (auto& e : ctx->pipe_ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  uint8_t* base = static_cast<uint8_t*>(ctx->io);
  uint32_t* d_w = reinterpret_cast<uint32_t*>(base);
  uint32_t* d_x = reinterpret_cast<uint32_t*>(base + w_b);
  uint8_t* d_y = base + w_b + x_b;
  double* d_sw = reinterpret_cast<double*>(base + w_b + x_b + y_b);
  double* d_sx = reinterpret_cast<double*>(base + w_b + x_b + y_b + sw_b);
  // row blocks: multiples of 256 rows, ~8 MB of output each, at most kPipeBlocks
  const uint64_t out_row_bytes = rows_x * 4;
  uint64_t blk = rows_w;
  if (rows_w * out_row_bytes > (16ull << 20) && rows_w >= 512) {
    blk = round_up(std::max<uint64_t>((8ull << 20) / out_row_bytes, 256), 256);
    blk = std::max<uint64_t>(blk, round_up((rows_w + kPipeBlocks - 1) / kPipeBlocks, 256));
    if (blk > rows_w) blk = rows_w;
  }
  const uint64_t nblk = (rows_w + blk - 1) / blk;
  const cudaStream_t sc = ctx->stream;
  // features (and scales) first, on the input copy stream
  CU(cudaMemcpyAsync(d_x, x, x_words * 4, cudaMemcpyHostToDevice, ctx->s_in));
  if (yf) {
    CU(cudaMemcpyAsync(d_sw, s_w, sw_n * 8, cudaMemcpyHostToDevice, ctx->s_in));
    CU(cudaMemcpyAsync(d_sx, s_x, sx_n * 8, cudaMemcpyHostToDevice, ctx->s_in));
  }
  for (uint64_t bi = 0; bi < nblk; ++bi) {
    const uint64_t r0 = bi * blk, rb = std::min(blk, rows_w - r0);
    // block bi's planes -> a packed buffer of rb rows ([plane][rb][wpr]) at d_w + n_w*r0*wpr
    uint32_t* d_wb = d_w + uint64_t(n_w) * r0 * wpr;
    CU(cudaMemcpy2DAsync(d_wb, rb * wpr * 4, w + r0 * wpr, rows_w * wpr * 4, rb * wpr * 4, n_w,
                         cudaMemcpyHostToDevice, ctx->s_in));
    cudaEvent_t ev_in = ctx->pipe_ev[(2 * bi) % (2 * kPipeBlocks)];
    cudaEvent_t ev_done = ctx->pipe_ev[(2 * bi + 1) % (2 * kPipeBlocks)];
    CU(cudaEventRecord(ev_in, ctx->s_in));
    CU(cudaStreamWaitEvent(sc, ev_in, 0));
    void* d_yb = d_y + r0 * out_row_bytes;
    st = run_matmul(ctx, d_wb, rb, n_w, yf ? d_sw + (gran_w == APMM_PER_ROW ? r0 : 0) : nullptr,
                    gran_w, d_x, rows_x, n_x, d_sx, gran_x, k,
                    yf ? nullptr : static_cast<int32_t*>(d_yb), yf ? static_cast<float*>(d_yb) : nullptr,
                    sc);
    if (st) return st;
    CU(cudaEventRecord(ev_done, sc));
    CU(cudaStreamWaitEvent(ctx->s_out, ev_done, 0));
    uint8_t* h_y = yf ? reinterpret_cast<uint8_t*>(yf) : reinterpret_cast<uint8_t*>(y);
    CU(cudaMemcpyAsync(h_y + r0 * out_row_bytes, d_yb, rb * out_row_bytes, cudaMemcpyDeviceToHost,
                       ctx->s_out));
  }
  CU(cudaStreamSynchronize(ctx->s_out));
  CU(cudaStreamSynchronize(sc));
  return APMM_OK;
}

int apmm_compute_plane_products(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w,
                                int n_w, const uint32_t* x_planes, uint64_t rows_x, int n_x,
                                uint64_t k, int32_t* stack) {
  int st;
  if (!ctx || !w_planes || !x_planes || !stack) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  if ((st = check_dims(rows_w, k, "weights")) || (st = check_dims(rows_x, k, "features"))) return st;
  if ((st = check_padding(w_planes, rows_w, k, n_w)) || (st = check_padding(x_planes, rows_x, k, n_x))) {
    return st;
  }
  if ((st = check_matmul(1, 1, rows_w, rows_x, k))) return st;
  const size_t w_words = apmm_packed_words(n_w, rows_w, k), x_words = apmm_packed_words(n_x, rows_x, k);
  const size_t w_b = align_up(w_words * 4), x_b = align_up(x_words * 4);
  const size_t s_n = size_t(n_w) * n_x * rows_w * rows_x;
  if ((st = ensure(&ctx->io, &ctx->io_bytes, w_b + x_b + align_up(s_n * 4), ctx->device))) return st;
  CU(cudaSetDevice(ctx->device));
  uint8_t* base = static_cast<uint8_t*>(ctx->io);
  uint32_t* d_w = reinterpret_cast<uint32_t*>(base);
  uint32_t* d_x = reinterpret_cast<uint32_t*>(base + w_b);
  int32_t* d_s = reinterpret_cast<int32_t*>(base + w_b + x_b);
  CU(cudaMemcpyAsync(d_w, w_planes, w_words * 4, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(d_x, x_planes, x_words * 4, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = apmm_cu_compute_plane_products(ctx, d_w, rows_w, n_w, d_x, rows_x, n_x, k, d_s,
                                            reinterpret_cast<apmm_stream_t>(ctx->stream)))) {
    return st;
  }
  CU(cudaMemcpyAsync(stack, d_s, s_n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return APMM_OK;
}

int apmm_recover(apmm_ctx* ctx, const int32_t* stack, int n_w, int n_x, uint64_t k,
                 uint64_t rows, uint64_t cols, int32_t* y) {
  int st;
  if (!ctx || !stack || !y) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  const size_t s_n = size_t(n_w) * n_x * rows * cols;
  const size_t s_b = align_up(s_n * 4);
  if ((st = ensure(&ctx->io, &ctx->io_bytes, s_b + align_up(rows * cols * 4), ctx->device))) return st;
  CU(cudaSetDevice(ctx->device));
  int32_t* d_s = static_cast<int32_t*>(ctx->io);
  int32_t* d_y = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(ctx->io) + s_b);
  CU(cudaMemcpyAsync(d_s, stack, s_n * 4, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = apmm_cu_recover(ctx, d_s, n_w, n_x, k, rows, cols, d_y,
                            reinterpret_cast<apmm_stream_t>(ctx->stream)))) {
    return st;
  }
  CU(cudaMemcpyAsync(y, d_y, rows * cols * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return APMM_OK;
}

int apmm_matmul_ap(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                   const uint32_t* x_planes, uint64_t rows_x, int n_x, uint64_t k, int32_t* y) {
  if (!ctx || !w_planes || !x_planes || !y) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  return host_matmul(ctx, w_planes, rows_w, n_w, nullptr, 0, x_planes, rows_x, n_x, nullptr, 0, k,
                     y, nullptr);
}

int apmm_matmul_ap_dequant(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                           const double* w_scales, int w_granularity, const uint32_t* x_planes,
                           uint64_t rows_x, int n_x, const double* x_scales, int x_granularity,
                           uint64_t k, float* out) {
  if (!ctx || !w_planes || !x_planes || !out || !w_scales || !x_scales) {
    return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  }
  if (!valid_gran(w_granularity) || !valid_gran(x_granularity)) {
    return fail(APMM_E_INVALID_ARGUMENT, "bad granularity");
  }
  return host_matmul(ctx, w_planes, rows_w, n_w, w_scales, w_granularity, x_planes, rows_x, n_x,
                     x_scales, x_granularity, k, nullptr, out);
}

}  // extern "C"
