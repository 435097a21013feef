// apmm_cuda.cu -- the C ABI (include/apmm_cuda.h): validation with the reference's error
// semantics, workspace management, and dispatch onto the sm_100a kernels.
//
// Validation order follows the reference so the same inputs fail with the same error
// class: BitWidth (bipolar.hpp:17-19) -> positive dimensions (bitplane.cpp:14-16) ->
// buffer contents (bitplane.cpp:22-32) -> K agreement / overflow_bound (kernel.cpp:189-199).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
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
  int route = APMM_ROUTE_AUTO;  // APMM_OPT_ROUTE
  bool early_w = true;          // APMM_OPT_EARLY_WEIGHT_READ
  bool early_x = false;         // APMM_OPT_EARLY_FEATURE_READ
  // stream binding (apmm_cuda.h, Conventions): the device entry points' stream
  bool bound = false;
  cudaStream_t bound_stream = nullptr;
  int host_depth = 0;  // > 0 inside a synchronous host entry point
  int ws_half = 0;  // which half of the ping-pong workspace the next matmul uses
  void* sk_ws = nullptr;  // K5 split-K accumulators (zero between calls)
  size_t sk_ws_bytes = 0;
  void* sk_scratch = nullptr;  // K5 feature fragments (ping-pong halves) + weight repack
  size_t sk_scratch_bytes = 0;
  void* tc_ws = nullptr;  // K6 feature codes + rowsum parts
  size_t tc_ws_bytes = 0;
  bool dbg_waits = false;  // APMM_DEBUG_WAITS=1: MMA-issuer wait-cycle counters (dev only)
  void* dbg = nullptr;  // APMM_DEBUG_WAITS counters (dev only)
  int* flags = nullptr;  // device error flags (recover: 2 ints; quantize / requant: 1)
  void* qx = nullptr;  // fused quantize: feature planes (skinny) / absmax + flag scratch
  size_t qx_bytes = 0;
  void* rq = nullptr;  // requant: absmax scratch (ordered u32 bits, rows_x + 1)
  size_t rq_bytes = 0;
  // dev launch trace (APMM_TRACE=<slots>, -DAPMM_DEVTOOLS builds only): per launch a slot of
  // [1024 CTAs][8] globaltimer stamps, round robin; trace_kind[slot] = kernel kind
  unsigned long long* trace = nullptr;
  int trace_slots = 0;
  int trace_seq = 0;
  std::vector<int> trace_kind;
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

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
}

// Grow a workspace buffer, stream-ordered on `s` (the only stream that uses it, by the
// context's stream binding): the old buffer is released with cudaFreeAsync after the work
// already enqueued on `s`, the new one comes from cudaMallocAsync -- no host or device-wide
// synchronisation. Growth inside a stream capture is refused (reserve first).
int ensure(void** buf, size_t* have, size_t need, int device, cudaStream_t s, bool zero = false) {
  if (need <= *have) return APMM_OK;
  if (capturing(s)) {
    return fail(APMM_E_INVALID_ARGUMENT,
                "workspace must grow from %zu to %zu bytes while the stream is being captured; "
                "call apmm_ctx_reserve with the largest shape before capturing",
                *have, need);
  }
  CU(cudaSetDevice(device));
  if (*buf) {
    CU(cudaFreeAsync(*buf, s));
    *buf = nullptr;
    *have = 0;
  }
  const size_t sz = need + need / 4;
  CU(cudaMallocAsync(buf, sz, s));
  if (zero) CU(cudaMemsetAsync(*buf, 0, sz, s));
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

// Kernel routes (apmm_cuda.h APMM_ROUTE_*). Every route computes the same bits.
enum class Route { Skinny, Mid, Pair, PairW, PairSplit, Single, StreamTc };

const char* route_name(Route r) {
  switch (r) {
    case Route::Skinny: return "skinny (K5)";
    case Route::Mid: return "mid split-K (K3f)";
    case Route::Pair: return "pair (K1 + K3)";
    case Route::PairW: return "pair weight-planes (K3f)";
    case Route::PairSplit: return "pair split-K (K1 + K3)";
    case Route::StreamTc: return "stream tensor-memory (K6)";
    default: return "single-SM (K1 + K3')";
  }
}

// Which routes can serve a call (their layout / output constraints).
struct RouteCaps {
  bool skinny, mid, pair_w, pair_split, stream_tc;
};
RouteCaps caps_of(const uint32_t* w, uint64_t rows_w, int n_w, uint64_t rows_x, uint64_t k,
                  const void* y, bool dequant, bool x_ready) {
  const bool splitk_out = !dequant && rows_x % 4 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0;
  RouteCaps c;
  c.skinny = rows_x <= kSkinnyMaxRowsX && !x_ready;
  c.mid = splitk_out && gemm_wplanes_addressable(w, k);
  c.pair_w = gemm_wplanes_addressable(w, k);
  c.pair_split = splitk_out;
  c.stream_tc = !dequant && !x_ready && stream_tc_supported(w, rows_w, rows_x, k, n_w, y);
  return c;
}

// AUTO. CTA-pair 256x256 tiles (K3) when they fill the machine. Otherwise mid-size calls
// (M_tok <= 256) take the split-K K3f: the weight planes are expanded on chip (each W row
// once: a single N tile), rowsum(U_w) formed by the transform warps, K split across CTA
// pairs, int32 partials TMA reduce-added into a Y zeroed by K1 (4096x128x4096 W2A4: 14.0 us
// vs 18.3 us for K1 + the 1-SM GEMM; profiles/r01b_mid_size_v2.txt). Feature counts up to
// kSkinnyPreferRows stay on K5 (faster there: 4096x40x4096 8.6 vs 12.6 us,
// profiles/r01b_skinny_mid_boundary.txt), and K5 takes up to 63 rows when the split-K path
// cannot (int32 output with a TMA-storable Y only). TENSOR_CORE = the same without K5.
// K6 (weight planes streamed into TMEM, tcgen05) for 16..128 feature rows (when it can serve:
// int32 output, rows_x % 4 == 0, n_w <= 4): 8192^2 W3A8 M = 16 / 32 / 64: 14.3 / 14.6 / 15.9 us
// vs 16.3 (K5) / 24.8 (K5) / 30.9 (K3f split-K); Llama-2-7B W2A4 M = 128: 4096x4096 12.3 vs
// 12.8, 11008x4096 17.7 vs 29.0, 4096x11008 17.7 vs 24.0 us (K3f)
// (profiles/r02/final/route_sweep.txt, profiles/r02/r2_k6_m128.txt). K5 stays faster below
// (M = 8: 11.5 vs 14.2 us; up to 15 rows K5 keeps two 8-column n-tiles).
constexpr uint64_t kStreamTcMinRows = 16;
constexpr uint64_t kStreamTcMaxRows = 128;

int pick_route(const apmm_ctx* ctx, const RouteCaps& c, uint64_t rows_w, uint64_t rows_x,
               Route* out) {
  const uint64_t pair_tiles = ((rows_w + 255) / 256) * ((rows_x + kPairN - 1) / kPairN);
  const bool pair = pair_tiles >= static_cast<uint64_t>(ctx->num_sms / 2);
  // K3f split-K up to 512 feature rows when the pair tiles cannot fill the machine:
  // 4096 x 384 / 512 x 4096 W2A4 21.0 / 21.8 us vs 23.5 / 22.3 (1-SM), 4096 x 384 / 512 x 11008
  // 44.0 / 44.9 vs 50.2 / 49.2 (profiles/r02/r2_route_sweep_m192_512.txt)
  const bool mid = c.mid && !pair && rows_x <= 512;
  auto forced = [&](bool ok, Route r) {
    if (!ok) {
      return fail(APMM_E_INVALID_ARGUMENT, "forced route %s cannot serve this call "
                  "(%llu x %llu)", route_name(r), (unsigned long long)rows_w,
                  (unsigned long long)rows_x);
    }
    *out = r;
    return int(APMM_OK);
  };
  switch (ctx->route) {
    case APMM_ROUTE_SKINNY: return forced(c.skinny, Route::Skinny);
    case APMM_ROUTE_MID_SPLITK: return forced(c.mid, Route::Mid);
    case APMM_ROUTE_PAIR: return forced(true, Route::Pair);
    case APMM_ROUTE_PAIR_WPLANES: return forced(c.pair_w, Route::PairW);
    case APMM_ROUTE_PAIR_SPLITK: return forced(c.pair_split, Route::PairSplit);
    case APMM_ROUTE_SINGLE_SM: return forced(true, Route::Single);
    case APMM_ROUTE_STREAM_TC: return forced(c.stream_tc, Route::StreamTc);
    default: break;
  }
  const bool allow_skinny = ctx->route != APMM_ROUTE_TENSOR_CORE;
  if (c.stream_tc && rows_x >= kStreamTcMinRows && rows_x <= kStreamTcMaxRows) {
    *out = Route::StreamTc;
  } else if (allow_skinny && c.skinny && (rows_x <= kSkinnyPreferRows || !mid)) {
    *out = Route::Skinny;
  } else if (pair) {
    *out = Route::Pair;
  } else if (mid) {
    *out = Route::Mid;
  } else {
    *out = Route::Single;
  }
  return APMM_OK;
}

// bytes 48..63: the split-K weight-plane GEMM's grid barrier (count, generation)
unsigned long long* grid_barrier(apmm_ctx* ctx) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ctx->flags) + 48);
}

// dev launch trace: the next slot (kind 1 expand, 2 pair GEMM, 3 weight-plane GEMM, 5 skinny)
unsigned long long* trace_slot(apmm_ctx* ctx, int kind) {
  if (!ctx->trace) return nullptr;
  const int slot = ctx->trace_seq++ % ctx->trace_slots;
  ctx->trace_kind[slot] = kind;
  return ctx->trace + uint64_t(slot) * 1024 * 8;
}

// blocks per SM of an expansion launch that runs after the previous kernel completed
// (6 x 128 threads x 80 registers = 61440 <= 64K: one wave on every SM)
constexpr int kK1xBlocksPerSm = 6;

// requant absmax scratch: rows_x u32 (+ 1 for the global max), 16-byte multiple (K1 zeroes it)
uint64_t colmax_bytes(uint64_t rows_x) { return round_up((rows_x + 1) * 4, 16); }

// Workspace a route needs for a call (growth is stream-ordered; see ensure()).
int reserve_skinny(apmm_ctx* ctx, uint64_t rows_w, uint64_t rows_x, uint64_t k, int n_w,
                   const void* w, cudaStream_t s) {
  int st = ensure(&ctx->sk_ws, &ctx->sk_ws_bytes, skinny_acc_bytes(rows_w, rows_x), ctx->device,
                  s, /*zero=*/true);  // split-K accumulators: zero at rest
  if (st) return st;
  return ensure(&ctx->sk_scratch, &ctx->sk_scratch_bytes,
                skinny_scratch_bytes(rows_w, rows_x, k, n_w, w), ctx->device, s);
}

// x_ready: the feature operand is already in this call's workspace half as u8 codes +
// rowsum (written by the fused quantize, K2 -> K3); then K1 expands W only and x is unused.
// colmax (dequant only): per-column absmax of the f32 output (requant), or null.
int run_matmul(apmm_ctx* ctx, const uint32_t* w, uint64_t rows_w, int n_w, const double* s_w,
               int gran_w, const uint32_t* x, uint64_t rows_x, int n_x, const double* s_x,
               int gran_x, uint64_t k, int32_t* y, float* yf, cudaStream_t stream,
               bool x_ready = false, unsigned* colmax = nullptr, bool colmax_global = false) {
  CU(cudaSetDevice(ctx->device));
  const RouteCaps caps = caps_of(w, rows_w, n_w, rows_x, k, yf ? static_cast<const void*>(yf) : y,
                                 yf != nullptr, x_ready);
  Route route;
  int st = pick_route(ctx, caps, rows_w, rows_x, &route);
  if (st) return st;
  if (route == Route::Skinny) {
    // few feature rows: feature prep + K5, the weight planes streamed once from HBM
    if ((st = reserve_skinny(ctx, rows_w, rows_x, k, n_w, w, stream))) return st;
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
    s.early_w = ctx->early_w;
    s.early_x = ctx->early_w && ctx->early_x;
    s.trace = trace_slot(ctx, 5);
    ctx->ws_half ^= 1;
    {
      // kernel timing brackets the streaming kernel alone (not the feature-prep launch)
      TimedLaunch t(ctx, 0, stream, /*record=*/false);
      s.ev_start = t.ev.first;
      s.ev_stop = t.ev.second;
      s.ev_flags = t.flags;
      CU(launch_skinny(s, stream));
    }
    ctx->launches += skinny_launches(rows_x);  // (feature prep +) streaming kernel
    if (colmax) {  // K5's epilogue does not form the column absmax: one pass over yf
      CU(cudaMemsetAsync(colmax, 0, colmax_bytes(rows_x), stream));
      CU(launch_colmax(yf, rows_w, rows_x, colmax, colmax_global, ctx->num_sms, stream));
      ctx->launches += 1;
    }
    return APMM_OK;
  }
  if (route == Route::StreamTc) {
    // feature prep (codes + rowsum, Y zeroed) + K6, the weight planes streamed once into TMEM
    if ((st = ensure(&ctx->tc_ws, &ctx->tc_ws_bytes,
                     stream_tc_ws_bytes(rows_x, k, rows_w, stream_tc_padded(rows_x, y)), ctx->device,
                     stream))) {
      return st;
    }
    StreamTcArgs s{};
    s.w_planes = w;
    s.x_planes = x;
    s.rows_w = rows_w;
    s.rows_x = rows_x;
    s.k = k;
    s.n_w = n_w;
    s.n_x = n_x;
    s.y = y;
    s.num_sms = ctx->num_sms;
    s.ws = ctx->tc_ws;
    s.early_w = ctx->early_w;
    s.early_x = ctx->early_w && ctx->early_x;
    s.trace_prep = trace_slot(ctx, 7);
    s.trace = trace_slot(ctx, 6);
    {
      TimedLaunch t(ctx, 0, stream, /*record=*/false);
      s.ev_start = t.ev.first;
      s.ev_stop = t.ev.second;
      s.ev_flags = t.flags;
      CU(launch_stream_tc(s, stream));
    }
    ctx->launches += stream_tc_padded(rows_x, y) ? 3 : 2;  // feature prep + K6 (+ unpad copy)
    return APMM_OK;
  }
  if ((st = ensure(&ctx->ws, &ctx->ws_bytes, matmul_ws_bytes(rows_w, rows_x, k), ctx->device,
                   stream))) {
    return st;
  }
  const MatmulWs m = carve(ctx->ws, rows_w, rows_x, k, ctx->ws_half);
  ctx->ws_half ^= 1;
  const uint64_t rsx_pad = round_up(rows_x, kRowsumPad);
  const bool wplanes = route == Route::Mid || route == Route::PairW;  // K3f expands W on chip
  const bool zero_y = route == Route::Mid || route == Route::PairSplit;  // split-K reduce-adds
  // the mid route expands its features and zeroes Y itself (in-kernel prep + grid barrier):
  // no K1 launch at all (the K1x launch + gap cost ~3 us of a ~12 us call, r02 notes)
  const bool xprep = route == Route::Mid && !x_ready;
  if (!xprep) {
    TimedLaunch t(ctx, 1, stream);
    // K1. K3f: W untouched except for rowsum(U_w) on the pair route (the split-K mid route
    // forms it in the GEMM); split-K: K1 also zeroes Y, which the units reduce-add into.
    // Work that must wait for the previous kernel (features unless the caller allows early
    // reads, the zeroing) runs in a second launch with the whole machine (K1x) when there
    // is also early work (weights) for a first, GEMM-co-resident launch (K1w).
    const uint64_t w_rows = route == Route::Mid ? 0 : rows_w;
    const bool early_x = ctx->early_w && ctx->early_x;
    void* zero_ptr = zero_y ? static_cast<void*>(y) : static_cast<void*>(colmax);
    const uint64_t zero_bytes = zero_y ? rows_w * rows_x * 4 : (colmax ? colmax_bytes(rows_x) : 0);
    const uint64_t x_rows = x_ready ? 0 : rows_x;
    const bool split_x = ctx->early_w && w_rows > 0 && !early_x && (x_rows > 0 || zero_bytes > 0);
    if (split_x) {
      CU(launch_expand(w, w_rows, n_w, wplanes ? nullptr : m.codes_w, m.rowsum_w, nullptr, 0,
                       x_ready ? 0 : rsx_pad, n_x, m.codes_x, m.rowsum_x, k, m.kpad,
                       ctx->num_sms, stream, nullptr, 0, true, false, trace_slot(ctx, 1)));
      CU(launch_expand(w, 0, n_w, nullptr, m.rowsum_w, x_ready ? nullptr : x, x_rows,
                       x_ready ? 0 : rsx_pad, n_x, m.codes_x, m.rowsum_x, k, m.kpad,
                       ctx->num_sms, stream, zero_ptr, zero_bytes, false, false,
                       trace_slot(ctx, 1), kK1xBlocksPerSm));
      ctx->launches += 1;
    } else {
      CU(launch_expand(w, w_rows, n_w, wplanes ? nullptr : m.codes_w, m.rowsum_w,
                       x_ready ? nullptr : x, x_rows, x_ready ? 0 : rsx_pad, n_x, m.codes_x,
                       m.rowsum_x, k, m.kpad, ctx->num_sms, stream, zero_ptr, zero_bytes,
                       ctx->early_w, early_x, trace_slot(ctx, 1),
                       w_rows == 0 || !ctx->early_w ? kK1xBlocksPerSm : 1));
    }
    ctx->launches += 1;
  }
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
  a.trace = route == Route::Single ? nullptr
                                    : trace_slot(ctx, route == Route::Mid || route == Route::PairW ? 3 : 2);
  // dev A/B (APMM_COLMAX_PASS=1): the absmax as a separate pass over yf on every route
  static const bool colmax_pass = APMM_DEV_ENV("APMM_COLMAX_PASS") != nullptr;
  const bool epi_colmax = route != Route::PairW && !colmax_pass;
  a.colmax = epi_colmax ? colmax : nullptr;
  a.early_w = ctx->early_w;
  if (xprep) {
    a.xprep_planes = x;
    a.xprep_rows_pad = rsx_pad;
    a.grid_bar = grid_barrier(ctx);
  }
  a.colmax_global = colmax_global;
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
    switch (route) {
      case Route::Mid: CU(launch_gemm_pair_wplanes(a, w, stream, &launches, /*split_k=*/true)); break;
      case Route::PairW: CU(launch_gemm_pair_wplanes(a, w, stream, &launches, false)); break;
      case Route::Pair: CU(launch_gemm_pair(a, stream, &launches, false)); break;
      case Route::PairSplit: CU(launch_gemm_pair(a, stream, &launches, /*split_k=*/true)); break;
      default: CU(launch_gemm_tc(a, stream, &launches)); break;
    }
  }
  ctx->launches += static_cast<uint64_t>(launches);
  if (colmax && !epi_colmax) {  // K3f's epilogue does not form the column absmax
    CU(launch_colmax(yf, rows_w, rows_x, colmax, colmax_global, ctx->num_sms, stream));
    ctx->launches += 1;
  }
  return APMM_OK;
}

// Device entry points run on exactly the stream they are given (NULL = the legacy default
// stream, as everywhere in CUDA), which must be the context's bound stream: the workspace
// is shared by every call of the context, so two streams would race on it
// (apmm_cuda.h, Conventions). The first device call binds; the host entry points run on
// ctx->stream after draining the bound stream, and skip the check for their inner calls.
int bind(apmm_ctx* ctx, apmm_stream_t st, cudaStream_t* out) {
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(st);
  *out = s;
  if (ctx->host_depth > 0) return APMM_OK;
  if (!ctx->bound) {
    ctx->bound = true;
    ctx->bound_stream = s;
    return APMM_OK;
  }
  if (ctx->bound_stream != s) {
    return fail(APMM_E_INVALID_ARGUMENT,
                "context is bound to stream %p but was called on stream %p: use one context per "
                "stream, or rebind with apmm_ctx_set_stream once the old stream's work is ordered",
                static_cast<void*>(ctx->bound_stream), static_cast<void*>(s));
  }
  return APMM_OK;
}

// Scope of a synchronous host entry point: drains device work enqueued on the bound stream
// (it shares the workspace) and runs the inner device calls on ctx->stream.
struct HostCall {
  apmm_ctx* ctx;
  int status = APMM_OK;
  explicit HostCall(apmm_ctx* c) : ctx(c) {
    if (!ctx) return;
    ++ctx->host_depth;
    cudaSetDevice(ctx->device);
    if (ctx->bound && ctx->bound_stream != ctx->stream) {
      const cudaError_t e = cudaStreamSynchronize(ctx->bound_stream);
      if (e != cudaSuccess) status = cuda_fail(e, "cudaStreamSynchronize(bound stream)");
    }
  }
  ~HostCall() {
    if (ctx) --ctx->host_depth;
  }
};

#define HOST_CALL(ctx)                          \
  HostCall host_call_(ctx);                     \
  if (host_call_.status) return host_call_.status

// Small per-context device scratch (ctx->flags, 64 bytes, zeroed at creation): [0..1]
// recover flags, [2] quantize non-finite flag, bytes 32..39 the per-tensor absmax bits,
// bytes 48..63 the grid barrier (count, generation).
int* quant_flag(apmm_ctx* ctx) { return ctx->flags + 2; }
unsigned long long* quant_amax(apmm_ctx* ctx) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(ctx->flags) + 32);
}


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
  if (const char* f = APMM_DEV_ENV("APMM_DEBUG_WAITS")) ctx->dbg_waits = f[0] == '1';
  if (const char* f = APMM_DEV_ENV("APMM_TRACE")) {
    ctx->trace_slots = std::max(1, std::atoi(f));
    const size_t b = size_t(ctx->trace_slots) * 1024 * 8 * 8;
    if (cudaMalloc(&ctx->trace, b) != cudaSuccess || cudaMemset(ctx->trace, 0, b) != cudaSuccess) {
      ctx->trace = nullptr;
    }
    ctx->trace_kind.assign(ctx->trace_slots, 0);
  }
  cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->flags, 64);
  if (e == cudaSuccess) e = cudaMemset(ctx->flags, 0, 64);  // incl. the grid-barrier counter
  if (e != cudaSuccess) {
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return cuda_fail(e, "context setup");
  }
  ctx->own_stream = true;
  *out = ctx;
  return APMM_OK;
}

int apmm_ctx_destroy(apmm_ctx* ctx) {
  if (!ctx) return APMM_OK;
  cudaSetDevice(ctx->device);
  // the context's work is on its bound stream and its own streams
  if (ctx->bound) cudaStreamSynchronize(ctx->bound_stream);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
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
  if (ctx->rq) cudaFree(ctx->rq);
  if (ctx->trace) cudaFree(ctx->trace);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->sk_ws) cudaFree(ctx->sk_ws);
  if (ctx->sk_scratch) cudaFree(ctx->sk_scratch);
  if (ctx->tc_ws) cudaFree(ctx->tc_ws);
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
  CU(cudaSetDevice(ctx->device));
  if (ctx->own_stream && ctx->stream) {
    CU(cudaStreamSynchronize(ctx->stream));
    cudaStreamDestroy(ctx->stream);
  }
  ctx->stream = reinterpret_cast<cudaStream_t>(stream);
  ctx->own_stream = false;
  ctx->bound = true;
  ctx->bound_stream = ctx->stream;
  return APMM_OK;
}

int apmm_ctx_set_option(apmm_ctx* ctx, int option, int value) {
  if (!ctx) return fail(APMM_E_INVALID_ARGUMENT, "null context");
  switch (option) {
    case APMM_OPT_ROUTE:
      if (value < APMM_ROUTE_AUTO || value > APMM_ROUTE_STREAM_TC) {
        return fail(APMM_E_INVALID_ARGUMENT, "unknown route %d", value);
      }
      ctx->route = value;
      return APMM_OK;
    case APMM_OPT_EARLY_WEIGHT_READ:
      ctx->early_w = value != 0;
      return APMM_OK;
    case APMM_OPT_EARLY_FEATURE_READ:
      ctx->early_x = value != 0;
      return APMM_OK;
    default:
      return fail(APMM_E_INVALID_ARGUMENT, "unknown option %d", option);
  }
}

int apmm_ctx_get_option(const apmm_ctx* ctx, int option, int* value) {
  if (!ctx || !value) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  switch (option) {
    case APMM_OPT_ROUTE: *value = ctx->route; return APMM_OK;
    case APMM_OPT_EARLY_WEIGHT_READ: *value = ctx->early_w ? 1 : 0; return APMM_OK;
    case APMM_OPT_EARLY_FEATURE_READ: *value = ctx->early_x ? 1 : 0; return APMM_OK;
    default: return fail(APMM_E_INVALID_ARGUMENT, "unknown option %d", option);
  }
}

int apmm_ctx_reserve(apmm_ctx* ctx, uint64_t rows_w, uint64_t rows_x, uint64_t k, int n_w) {
  int st;
  if (!ctx) return fail(APMM_E_INVALID_ARGUMENT, "null context");
  if ((st = check_width(n_w)) || (st = check_dims(rows_w, k, "weights")) ||
      (st = check_dims(rows_x, k, "features"))) {
    return st;
  }
  const cudaStream_t s = ctx->bound ? ctx->bound_stream : ctx->stream;
  if ((st = ensure(&ctx->ws, &ctx->ws_bytes, matmul_ws_bytes(rows_w, rows_x, k), ctx->device, s))) {
    return st;
  }
  if ((st = ensure(&ctx->tc_ws, &ctx->tc_ws_bytes,
                   stream_tc_ws_bytes(rows_x, k, rows_w, rows_x <= kStreamTcMaxRows), ctx->device, s))) {
    return st;
  }
  if (rows_x <= kSkinnyMaxRowsX) {
    // worst case: a weight buffer that needs the 16-byte repack
    if ((st = reserve_skinny(ctx, rows_w, rows_x, k, n_w, reinterpret_cast<const void*>(4), s))) {
      return st;
    }
  }
  if ((st = ensure(&ctx->qx, &ctx->qx_bytes, apmm_packed_words(8, rows_x, k) * 4 + 64, ctx->device,
                   s))) {
    return st;
  }
  if ((st = ensure(&ctx->rq, &ctx->rq_bytes, (rows_x + 1) * 4, ctx->device, s))) return st;
  CU(cudaStreamSynchronize(s));
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
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
  CU(launch_pack(codes, rows, cols, n, planes, s));
  ctx->launches += 1;
  return APMM_OK;
}

int apmm_cu_unpack(apmm_ctx* ctx, const uint32_t* planes, uint64_t rows, uint64_t cols, int n,
                   uint8_t* codes, apmm_stream_t stream) {
  int st;
  if (!ctx || !codes || !planes) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "PackedBitPlanes"))) return st;
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
  CU(launch_unpack(planes, rows, cols, n, codes, s));
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
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
  unsigned long long* amax = quant_amax(ctx);
  int* flag = quant_flag(ctx);
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
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  return run_matmul(ctx, w_planes, rows_w, n_w, nullptr, 0, x_planes, rows_x, n_x, nullptr, 0, k,
                    y, nullptr, s);
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
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  return run_matmul(ctx, w_planes, rows_w, n_w, w_scales, w_granularity, x_planes, rows_x, n_x,
                    x_scales, x_granularity, k, nullptr, out, s);
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
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  const uint64_t wpr = (k + 31) / 32;
  return run_matmul(ctx, w_planes + uint64_t(weight_plane) * rows_w * wpr, rows_w, 1, nullptr, 0,
                    x_planes + uint64_t(feature_plane) * rows_x * wpr, rows_x, 1, nullptr, 0, k,
                    y, nullptr, s);
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
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
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
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
  if (rows_x <= kSkinnyMaxRowsX && ctx->route != APMM_ROUTE_TENSOR_CORE &&
      (ctx->route == APMM_ROUTE_AUTO || ctx->route == APMM_ROUTE_SKINNY)) {
    // few feature rows: the skinny kernel consumes planes -> quantize_pack into a scratch
    // plane buffer, then the ordinary device matmul (both stream-ordered)
    const size_t words = apmm_packed_words(n_x, rows_x, k);
    if ((st = ensure(&ctx->qx, &ctx->qx_bytes, words * 4 + 64, ctx->device, s))) return st;
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
  if ((st = ensure(&ctx->ws, &ctx->ws_bytes, matmul_ws_bytes(rows_w, rows_x, k), ctx->device,
                   s))) {
    return st;
  }
  const MatmulWs m = carve(ctx->ws, rows_w, rows_x, k, ctx->ws_half);
  unsigned long long* amax = quant_amax(ctx);
  int* flag = quant_flag(ctx);
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

int apmm_cu_dot_1bit_xor(apmm_ctx* ctx, const uint32_t* a, uint64_t a_words, const uint32_t* b,
                         uint64_t b_words, uint64_t k, int64_t* out, apmm_stream_t stream) {
  if (!ctx || !a || !b || !out) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  // kernel.cpp:117-121, same order and messages
  if (k == 0) return fail(APMM_E_OUT_OF_RANGE, "k_logical must be positive");
  const uint64_t need = (k + 31) / 32;
  if (a_words != need || b_words != need) {
    return fail(APMM_E_LENGTH_MISMATCH, "word sequences must hold exactly ceil(k/32) words");
  }
  int st;
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
  CU(launch_dot_xor(a, b, need, k, out, s));
  ctx->launches += 1;
  return APMM_OK;
}

int apmm_cu_matmul_ap_requant(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                              const double* w_scales, int w_granularity, const uint32_t* x_planes,
                              uint64_t rows_x, int n_x, const double* x_scales, int x_granularity,
                              uint64_t k, int n_next, int next_granularity, float* yf,
                              uint32_t* next_planes, double* next_scales, double* absmax,
                              apmm_stream_t stream) {
  if (!ctx || !w_planes || !x_planes || !w_scales || !x_scales || !yf) {
    return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  }
  if (!absmax && (!next_planes || !next_scales)) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if (!valid_gran(w_granularity) || !valid_gran(x_granularity) || !valid_gran(next_granularity)) {
    return fail(APMM_E_INVALID_ARGUMENT, "bad granularity");
  }
  int st;
  if ((st = check_width(n_next))) return st;
  if ((st = check_matmul(n_w, n_x, rows_w, rows_x, k))) return st;
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
  if ((st = ensure(&ctx->rq, &ctx->rq_bytes, colmax_bytes(rows_x), ctx->device, s))) return st;
  const bool global = next_granularity == APMM_PER_TENSOR;
  unsigned* colmax = static_cast<unsigned*>(ctx->rq);
  if ((st = run_matmul(ctx, w_planes, rows_w, n_w, w_scales, w_granularity, x_planes, rows_x, n_x,
                       x_scales, x_granularity, k, nullptr, yf, s, false, colmax, global))) {
    return st;
  }
  if (absmax) {  // split form: hand out the local maxima (as doubles) for a cross-GPU max
    CU(launch_bits_to_double(colmax, global ? 1 : rows_x, absmax, s));
    ctx->launches += 1;
    return APMM_OK;
  }
  CU(cudaMemsetAsync(quant_flag(ctx), 0, sizeof(int), s));
  CU(launch_requant_pack(yf, rows_w, rows_x, colmax, global, n_next, next_planes, next_scales,
                         quant_flag(ctx), s));
  ctx->launches += 1;
  int h_flag = 0;  // the reference's quantize throws NonFinite (bipolar.cpp:73-75)
  CU(cudaMemcpyAsync(&h_flag, quant_flag(ctx), sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (h_flag) return fail(APMM_E_NON_FINITE, "input contains NaN or infinity");
  return APMM_OK;
}

int apmm_cu_requant_pack(apmm_ctx* ctx, const float* yf, uint64_t rows_w, uint64_t rows_x,
                         const double* absmax, int n_next, int next_granularity,
                         uint32_t* next_planes, double* next_scales, apmm_stream_t stream) {
  if (!ctx || !yf || !absmax || !next_planes || !next_scales) {
    return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  }
  if (!valid_gran(next_granularity)) return fail(APMM_E_INVALID_ARGUMENT, "bad granularity");
  int st;
  if ((st = check_width(n_next)) || (st = check_dims(rows_x, rows_w, "RealMatrix"))) return st;
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
  if ((st = ensure(&ctx->rq, &ctx->rq_bytes, colmax_bytes(rows_x), ctx->device, s))) return st;
  const bool global = next_granularity == APMM_PER_TENSOR;
  unsigned* colmax = static_cast<unsigned*>(ctx->rq);
  CU(launch_double_to_bits(absmax, global ? 1 : rows_x, colmax, s));
  CU(cudaMemsetAsync(quant_flag(ctx), 0, sizeof(int), s));
  CU(launch_requant_pack(yf, rows_w, rows_x, colmax, global, n_next, next_planes, next_scales,
                         quant_flag(ctx), s));
  ctx->launches += 2;
  int h_flag = 0;
  CU(cudaMemcpyAsync(&h_flag, quant_flag(ctx), sizeof(int), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (h_flag) return fail(APMM_E_NON_FINITE, "input contains NaN or infinity");
  return APMM_OK;
}

// ---- host entry points ------------------------------------------------------------------
int apmm_decompose_and_pack(apmm_ctx* ctx, const uint8_t* codes, uint64_t rows, uint64_t cols,
                            int n, uint32_t* planes) {
  int st;
  if (!ctx || !codes || !planes) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  HOST_CALL(ctx);
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "CodeMatrix"))) return st;
  const uint32_t limit = 1u << n;
  for (uint64_t e = 0; e < rows * cols; ++e) {  // CodeMatrix ctor (bipolar.cpp:33-36)
    if (codes[e] >= limit) return fail(APMM_E_OUT_OF_RANGE, "code has bits above position n-1");
  }
  const size_t in_b = align_up(rows * cols), out_b = apmm_packed_words(n, rows, cols) * 4;
  if ((st = ensure(&ctx->io, &ctx->io_bytes, in_b + out_b, ctx->device, ctx->stream))) return st;
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
  HOST_CALL(ctx);
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "PackedBitPlanes"))) return st;
  if ((st = check_padding(planes, rows, cols, n))) return st;
  const size_t in_b = align_up(apmm_packed_words(n, rows, cols) * 4), out_b = rows * cols;
  if ((st = ensure(&ctx->io, &ctx->io_bytes, in_b + out_b, ctx->device, ctx->stream))) return st;
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
  HOST_CALL(ctx);
  if (!valid_gran(granularity)) return fail(APMM_E_INVALID_ARGUMENT, "bad granularity");
  if ((st = check_width(n)) || (st = check_dims(rows, cols, "RealMatrix"))) return st;
  const uint64_t n_scales = granularity == APMM_PER_ROW ? rows : 1;
  const size_t x_b = align_up(rows * cols * 8), p_b = align_up(apmm_packed_words(n, rows, cols) * 4);
  const size_t s_b = align_up(n_scales * 8), c_b = align_up(rows * cols);
  if ((st = ensure(&ctx->io, &ctx->io_bytes, x_b + p_b + s_b + c_b, ctx->device, ctx->stream))) return st;
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
  HOST_CALL(ctx);
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
  if ((st = ensure(&ctx->io, &ctx->io_bytes, w_b + x_b + y_b + sw_b + sx_b, ctx->device, ctx->stream))) return st;
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
  HOST_CALL(ctx);
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  if ((st = check_dims(rows_w, k, "weights")) || (st = check_dims(rows_x, k, "features"))) return st;
  if ((st = check_padding(w_planes, rows_w, k, n_w)) || (st = check_padding(x_planes, rows_x, k, n_x))) {
    return st;
  }
  if ((st = check_matmul(1, 1, rows_w, rows_x, k))) return st;
  const size_t w_words = apmm_packed_words(n_w, rows_w, k), x_words = apmm_packed_words(n_x, rows_x, k);
  const size_t w_b = align_up(w_words * 4), x_b = align_up(x_words * 4);
  const size_t s_n = size_t(n_w) * n_x * rows_w * rows_x;
  if ((st = ensure(&ctx->io, &ctx->io_bytes, w_b + x_b + align_up(s_n * 4), ctx->device, ctx->stream))) return st;
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
  HOST_CALL(ctx);
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  const size_t s_n = size_t(n_w) * n_x * rows * cols;
  const size_t s_b = align_up(s_n * 4);
  if ((st = ensure(&ctx->io, &ctx->io_bytes, s_b + align_up(rows * cols * 4), ctx->device, ctx->stream))) return st;
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

int apmm_dot_1bit_xor(apmm_ctx* ctx, const uint32_t* a, uint64_t a_words, const uint32_t* b,
                      uint64_t b_words, uint64_t k, int64_t* out) {
  if (!ctx || !a || !b || !out) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if (k == 0) return fail(APMM_E_OUT_OF_RANGE, "k_logical must be positive");
  const uint64_t need = (k + 31) / 32;
  if (a_words != need || b_words != need) {
    return fail(APMM_E_LENGTH_MISMATCH, "word sequences must hold exactly ceil(k/32) words");
  }
  HOST_CALL(ctx);
  int st;
  const size_t w_b = align_up(need * 4);
  if ((st = ensure(&ctx->io, &ctx->io_bytes, 2 * w_b + 64, ctx->device, ctx->stream))) return st;
  uint8_t* base = static_cast<uint8_t*>(ctx->io);
  uint32_t* d_a = reinterpret_cast<uint32_t*>(base);
  uint32_t* d_b = reinterpret_cast<uint32_t*>(base + w_b);
  int64_t* d_o = reinterpret_cast<int64_t*>(base + 2 * w_b);
  CU(cudaMemcpyAsync(d_a, a, need * 4, cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(d_b, b, need * 4, cudaMemcpyHostToDevice, ctx->stream));
  if ((st = apmm_cu_dot_1bit_xor(ctx, d_a, need, d_b, need, k, d_o,
                                 reinterpret_cast<apmm_stream_t>(ctx->stream)))) {
    return st;
  }
  CU(cudaMemcpyAsync(out, d_o, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return APMM_OK;
}

int apmm_matmul_plane_pair(apmm_ctx* ctx, const uint32_t* w_planes, uint64_t rows_w, int n_w,
                           int weight_plane, const uint32_t* x_planes, uint64_t rows_x, int n_x,
                           int feature_plane, uint64_t k, int32_t* y) {
  int st;
  if (!ctx || !w_planes || !x_planes || !y) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  HOST_CALL(ctx);
  if ((st = check_width(n_w)) || (st = check_width(n_x))) return st;
  if ((st = check_dims(rows_w, k, "weights")) || (st = check_dims(rows_x, k, "features"))) return st;
  if ((st = check_padding(w_planes, rows_w, k, n_w)) || (st = check_padding(x_planes, rows_x, k, n_x))) {
    return st;
  }
  if (weight_plane < 0 || weight_plane >= n_w || feature_plane < 0 || feature_plane >= n_x) {
    return fail(APMM_E_INDEX_OUT_OF_BOUNDS, "plane pair (%d, %d) out of range", weight_plane,
                feature_plane);
  }
  const uint64_t wpr = (k + 31) / 32;
  const size_t w_b = align_up(rows_w * wpr * 4), x_b = align_up(rows_x * wpr * 4);
  if ((st = ensure(&ctx->io, &ctx->io_bytes, w_b + x_b + align_up(rows_w * rows_x * 4), ctx->device,
                   ctx->stream))) {
    return st;
  }
  uint8_t* base = static_cast<uint8_t*>(ctx->io);
  uint32_t* d_w = reinterpret_cast<uint32_t*>(base);
  uint32_t* d_x = reinterpret_cast<uint32_t*>(base + w_b);
  int32_t* d_y = reinterpret_cast<int32_t*>(base + w_b + x_b);
  // only the two planes travel (plane_row offsets, bitplane.cpp:44)
  CU(cudaMemcpyAsync(d_w, w_planes + uint64_t(weight_plane) * rows_w * wpr, rows_w * wpr * 4,
                     cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(d_x, x_planes + uint64_t(feature_plane) * rows_x * wpr, rows_x * wpr * 4,
                     cudaMemcpyHostToDevice, ctx->stream));
  if ((st = apmm_cu_matmul_plane_pair(ctx, d_w, rows_w, 1, 0, d_x, rows_x, 1, 0, k, d_y,
                                      reinterpret_cast<apmm_stream_t>(ctx->stream)))) {
    return st;
  }
  CU(cudaMemcpyAsync(y, d_y, rows_w * rows_x * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  return APMM_OK;
}

// ---- APMM v1 tensor files (tensor_file.hpp:12-64) --------------------------------------
static uint32_t rd_u32(const uint8_t* p) {
  return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}
static uint64_t rd_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= uint64_t(p[i]) << (8 * i);
  return v;
}

// parse_tensor (tensor_file.cpp:159-229): same checks, same order, same messages.
int apmm_tensor_parse(const uint8_t* bytes, uint64_t n, apmm_tensor_info* info) {
  if (!bytes || !info) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if (n < 16) return fail(APMM_E_PARSE, "truncated tensor header");
  if (std::memcmp(bytes, "APMM", 4) != 0) return fail(APMM_E_PARSE, "bad magic bytes");
  if (bytes[4] != 0x01) return fail(APMM_E_PARSE, "unsupported tensor version %d", int(bytes[4]));
  apmm_tensor_info t{};
  t.bit_width = bytes[6];
  const int gran = bytes[7];
  t.rows = rd_u32(bytes + 8);
  t.cols = rd_u32(bytes + 12);
  if (t.rows == 0 || t.cols == 0) return fail(APMM_E_PARSE, "tensor dimensions must be positive");
  const uint64_t elems = t.rows * t.cols;
  uint64_t off = 16;
  if (bytes[5] == 0x00) {
    t.kind = 0;
    t.granularity = -1;
    if (t.bit_width != 0) return fail(APMM_E_PARSE, "float tensor must carry bit width 0");
    if (gran != 0xFF) return fail(APMM_E_PARSE, "float tensor granularity must be 0xFF");
    if (n != off + elems * 4) {
      return fail(APMM_E_PARSE, "float payload length mismatch: file holds %llu bytes, expected %llu",
                  (unsigned long long)(n - off), (unsigned long long)(elems * 4));
    }
    t.payload_offset = off;
    t.payload_words = elems;
    *info = t;
    return APMM_OK;
  }
  if (bytes[5] != 0x01) return fail(APMM_E_PARSE, "unknown tensor kind %d", int(bytes[5]));
  t.kind = 1;
  if (t.bit_width < 1 || t.bit_width > 8) return fail(APMM_E_PARSE, "quantized bit width must be in [1, 8]");
  if (gran == 0x00) {
    t.scale_count = 1;
  } else if (gran == 0x01) {
    t.scale_count = t.rows;
  } else {
    return fail(APMM_E_PARSE, "quantized granularity must be 0x00 or 0x01");
  }
  t.granularity = gran;
  if (n < off + t.scale_count * 8) return fail(APMM_E_PARSE, "truncated scale block");
  for (uint64_t i = 0; i < t.scale_count; ++i) {
    const uint64_t b = rd_u64(bytes + off + i * 8);
    double v;
    std::memcpy(&v, &b, 8);
    if (!std::isfinite(v) || v <= 0.0) return fail(APMM_E_PARSE, "scales must be finite and positive");
  }
  off += t.scale_count * 8;
  const uint64_t words = apmm_packed_words(t.bit_width, t.rows, t.cols);
  if (n != off + words * 4) {
    return fail(APMM_E_PARSE, "packed payload length mismatch: file holds %llu bytes, expected %llu",
                (unsigned long long)(n - off), (unsigned long long)(words * 4));
  }
  t.payload_offset = off;
  t.payload_words = words;
  // to_packed -> PackedBitPlanes constructor: padding bits must be zero (bitplane.cpp:22-32)
  const uint32_t tail = static_cast<uint32_t>(t.cols & 31);
  if (tail) {
    const uint32_t pad = ~((1u << tail) - 1u);
    const uint64_t wpr = (t.cols + 31) / 32;
    for (uint64_t pr = 0; pr < uint64_t(t.bit_width) * t.rows; ++pr) {
      if (rd_u32(bytes + off + ((pr + 1) * wpr - 1) * 4) & pad) {
        return fail(APMM_E_OUT_OF_RANGE, "packed buffer has nonzero padding bits");
      }
    }
  }
  *info = t;
  return APMM_OK;
}

int apmm_cu_tensor_upload(apmm_ctx* ctx, const uint8_t* bytes, uint64_t n, uint32_t* planes,
                          double* scales, double* values, apmm_stream_t stream) {
  if (!ctx) return fail(APMM_E_INVALID_ARGUMENT, "null context");
  apmm_tensor_info t;
  int st = apmm_tensor_parse(bytes, n, &t);
  if (st) return st;
  cudaStream_t s;
  if ((st = bind(ctx, stream, &s))) return st;
  CU(cudaSetDevice(ctx->device));
  if (t.kind == 1) {
    // the payload IS the PackedBitPlanes buffer (tensor_file.cpp:218-228): one copy, no relayout
    if (planes) {
      CU(cudaMemcpyAsync(planes, bytes + t.payload_offset, t.payload_words * 4,
                         cudaMemcpyHostToDevice, s));
    }
    if (scales) {
      CU(cudaMemcpyAsync(scales, bytes + 16, t.scale_count * 8, cudaMemcpyHostToDevice, s));
    }
    return APMM_OK;
  }
  if (values) {  // f32 payload -> device staging -> widened to f64 on device (to_real)
    if ((st = ensure(&ctx->qx, &ctx->qx_bytes, t.payload_words * 4, ctx->device, s))) return st;
    CU(cudaMemcpyAsync(ctx->qx, bytes + t.payload_offset, t.payload_words * 4,
                       cudaMemcpyHostToDevice, s));
    CU(launch_widen(static_cast<const float*>(ctx->qx), t.payload_words, values, s));
    ctx->launches += 1;
  }
  return APMM_OK;
}

int apmm_tensor_file_load(apmm_ctx* ctx, const char* path, apmm_tensor_info* info,
                          uint32_t* planes, double* scales, double* values) {
  if (!ctx || !path) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  // read_tensor_file (tensor_file.cpp:231-): IoError when the file cannot be read
  FILE* f = std::fopen(path, "rb");
  if (!f) return fail(APMM_E_IO, "cannot open %s for reading", path);
  std::vector<uint8_t> bytes;
  uint8_t buf[1 << 16];
  size_t got;
  while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) bytes.insert(bytes.end(), buf, buf + got);
  const bool bad = std::ferror(f) != 0;
  std::fclose(f);
  if (bad) return fail(APMM_E_IO, "short read from %s", path);
  HOST_CALL(ctx);
  apmm_tensor_info t;
  int st = apmm_tensor_parse(bytes.data(), bytes.size(), &t);
  if (st) return st;
  if (info) *info = t;
  if ((st = apmm_cu_tensor_upload(ctx, bytes.data(), bytes.size(), planes, scales, values,
                                  reinterpret_cast<apmm_stream_t>(ctx->stream)))) {
    return st;
  }
  CU(cudaStreamSynchronize(ctx->stream));
  return APMM_OK;
}

// serialize_tensor (tensor_file.cpp:135-157) for the quantized kind, with the consistency
// checks of check_consistent (tensor_file.cpp:47-85).
int apmm_tensor_serialize_quantized(uint64_t rows, uint64_t cols, int n, int granularity,
                                    const double* scales, const uint32_t* planes, uint8_t* out,
                                    uint64_t out_cap, uint64_t* out_len) {
  if (!scales || !planes || !out_len) return fail(APMM_E_INVALID_ARGUMENT, "null argument");
  if (rows == 0 || cols == 0) return fail(APMM_E_OUT_OF_RANGE, "tensor dimensions must be positive");
  if (rows > 0xFFFFFFFFull || cols > 0xFFFFFFFFull) {
    return fail(APMM_E_OUT_OF_RANGE, "matrix too large for tensor file");
  }
  if (n < 1 || n > 8) return fail(APMM_E_OUT_OF_RANGE, "quantized bit width must be in [1, 8]");
  if (!valid_gran(granularity)) {
    return fail(APMM_E_OUT_OF_RANGE, "quantized granularity must be per-tensor or per-row");
  }
  const uint64_t sc = granularity == APMM_PER_ROW ? rows : 1;
  for (uint64_t i = 0; i < sc; ++i) {
    if (!std::isfinite(scales[i]) || scales[i] <= 0.0) {
      return fail(APMM_E_OUT_OF_RANGE, "scales must be finite and positive");
    }
  }
  const uint64_t words = apmm_packed_words(n, rows, cols);
  const uint64_t len = 16 + sc * 8 + words * 4;
  *out_len = len;
  if (!out) return APMM_OK;
  if (out_cap < len) return fail(APMM_E_LENGTH_MISMATCH, "output buffer holds %llu bytes, need %llu",
                                 (unsigned long long)out_cap, (unsigned long long)len);
  std::memcpy(out, "APMM", 4);
  out[4] = 0x01;
  out[5] = 0x01;
  out[6] = static_cast<uint8_t>(n);
  out[7] = static_cast<uint8_t>(granularity);
  for (int i = 0; i < 4; ++i) out[8 + i] = static_cast<uint8_t>(rows >> (8 * i));
  for (int i = 0; i < 4; ++i) out[12 + i] = static_cast<uint8_t>(cols >> (8 * i));
  uint8_t* p = out + 16;
  for (uint64_t i = 0; i < sc; ++i) {
    uint64_t b;
    std::memcpy(&b, &scales[i], 8);
    for (int j = 0; j < 8; ++j) *p++ = static_cast<uint8_t>(b >> (8 * j));
  }
  for (uint64_t w = 0; w < words; ++w) {
    for (int j = 0; j < 4; ++j) *p++ = static_cast<uint8_t>(planes[w] >> (8 * j));
  }
  return APMM_OK;
}

#ifdef APMM_DEVTOOLS
// dev only (not in the release .so): copy the launch trace out and clear it. out holds
// slots x 1024 x 8 u64, kinds `slots` ints; returns the number of launches recorded so far.
__attribute__((visibility("default"))) int apmm_dev_trace_read(apmm_ctx* ctx, unsigned long long* out,
                                                            int* kinds) {
  if (!ctx || !ctx->trace) return -1;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  const size_t b = size_t(ctx->trace_slots) * 1024 * 8 * 8;
  cudaMemcpy(out, ctx->trace, b, cudaMemcpyDeviceToHost);
  cudaMemset(ctx->trace, 0, b);
  for (int i = 0; i < ctx->trace_slots; ++i) kinds[i] = ctx->trace_kind[i];
  const int n = ctx->trace_seq;
  ctx->trace_seq = 0;
  return n;
}
#endif

}  // extern "C"
