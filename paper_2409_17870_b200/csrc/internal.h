// internal.h -- declarations shared by the .cu translation units of libapmm_b200.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

// Development instrumentation (plan dumps, per-phase CTA timelines, wait-cycle counters,
// ablations and route/stage overrides read from the environment) is compiled only with
// -DAPMM_DEVTOOLS (python -m paper_2409_17870_b200.build --dev). The release library never
// reads the environment: APMM_DEV_ENV is a null constant and the names are not in the .so.
#ifdef APMM_DEVTOOLS
#define APMM_DEV_ENV(name) std::getenv(name)
#else
#define APMM_DEV_ENV(name) (static_cast<const char*>(nullptr))
#endif

namespace apmm_b200 {

// cudaFuncSetAttribute and occupancy queries are per device; a process may drive several
// devices through several contexts. One bit / slot per device ordinal.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d & (kMaxDevices - 1);
}
struct DeviceBits {
  std::atomic<uint64_t> bits{0};
  bool test(int dev) const { return (bits.load(std::memory_order_acquire) >> dev) & 1u; }
  void set(int dev) { bits.fetch_or(uint64_t(1) << dev, std::memory_order_acq_rel); }
};

// Geometry of the tensor-core GEMM (gemm_tc.cu).
constexpr int kBM = 128;        // weight rows per CTA tile (MMA M, TMEM lanes)
constexpr int kBN = 256;        // feature rows per CTA tile (MMA N)
constexpr int kBK = 128;        // K bytes per pipeline stage (one 128-B swizzle row)
constexpr int kKAlign = kBK;    // device code rows are padded to a multiple of this
constexpr int kPairN = 256;     // feature rows per CTA-pair tile (gemm_pair.cu, MMA N)
constexpr int kRowsumPad = kBN; // rowsum_x is zero-padded to a multiple of this

inline uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

// Grouped tile raster for the persistent GEMMs: linear tile t -> (tm, tn) walking groups of
// kRasterGroup W row tiles across every X column tile. A wave of 74 pair tiles then covers
// ~8 W tiles x ~9 X tiles, so both operands' codes are reused from L2; with the plain
// "tm fastest" order a tall W (70B FFN: 112 row tiles, 235 MB of codes) was re-streamed
// from HBM once per X column tile.
constexpr uint32_t kRasterGroup = 8;
__host__ __device__ inline void raster_tile(uint32_t t, uint32_t tiles_m, uint32_t tiles_n,
                                            uint32_t& tm, uint32_t& tn) {
  const uint32_t per_group = kRasterGroup * tiles_n;
  const uint32_t g = t / per_group, first = g * kRasterGroup;
  const uint32_t gsize = tiles_m - first < kRasterGroup ? tiles_m - first : kRasterGroup;
  const uint32_t r = t - g * per_group;
  tm = first + r % gsize;
  tn = r / gsize;
}

// ---- prep.cu -------------------------------------------------------------------------
// Both operands' planes (reference layout) -> u8 codes [rows x kpad] (zero K padding, K
// permuted identically within each 32-column group) + rowsum[rows], one launch.
// rowsum_x[rows_x, rows_x_pad) is zeroed. Launched with PDL (see prep.cu). w_codes may be
// null: then only rowsum_w is produced for W (the fused GEMM expands W on chip); rows_w may
// be 0 (W untouched). zero_out[0, zero_bytes) (16-B multiple) is zeroed after the previous
// kernel in the stream completed (Y of a split-K GEMM).
// PDL: W rows are expanded before griddepcontrol.wait when early_w (weights may be read
// while the previous kernel in the stream drains), X rows too when early_x (caller's
// promise, APMM_OPT_EARLY_FEATURE_READ), the zeroing always after it.
cudaError_t launch_expand(const uint32_t* w_planes, uint64_t rows_w, int n_w,
                          uint8_t* w_codes, int32_t* w_rowsum, const uint32_t* x_planes,
                          uint64_t rows_x, uint64_t rows_x_pad, int n_x, uint8_t* x_codes,
                          int32_t* x_rowsum, uint64_t cols, uint64_t kpad, int num_sms,
                          cudaStream_t s, void* zero_out = nullptr, uint64_t zero_bytes = 0,
                          bool early_w = true, bool early_x = false,
                          unsigned long long* trace = nullptr, int blocks_per_sm = 1);
cudaError_t launch_pack(const uint8_t* codes, uint64_t rows, uint64_t cols, int n,
                        uint32_t* planes, cudaStream_t s);
cudaError_t launch_unpack(const uint32_t* planes, uint64_t rows, uint64_t cols, int n,
                          uint8_t* codes, cudaStream_t s);
// fp64 quantize + pack. flag[0] receives 1 if any input is non-finite. `amax_bits` is a
// scratch u64 (per-tensor absmax as ordered bits).
// With gemm_codes != null it also (or, with planes == null, only) writes the GEMM operand
// directly: u8 codes [rows][kpad] in K1's layout + rowsum[rows_pad] (zero padded) -- K2
// feeding K3 without the bit planes and the X expansion.
cudaError_t launch_quantize_pack(const double* x, uint64_t rows, uint64_t cols, int n,
                                 int granularity, uint32_t* planes, double* scales,
                                 uint8_t* codes, unsigned long long* amax_bits, int* flag,
                                 cudaStream_t s, uint8_t* gemm_codes = nullptr,
                                 int32_t* gemm_rowsum = nullptr, uint64_t kpad = 0,
                                 uint64_t rowsum_pad = 0);

// dot_1bit_xor (kernel.cpp:115-123) into *out (device int64), one block.
cudaError_t launch_dot_xor(const uint32_t* a, const uint32_t* b, uint64_t words, uint64_t k,
                           int64_t* out, cudaStream_t s);
// f32 -> f64 (tensor file float payload, to_real).
cudaError_t launch_widen(const float* src, uint64_t n, double* dst, cudaStream_t s);
// Column (per-token) or global absmax of yf [rows_w x rows_x] f32 as ordered u32 bits of |v|
// (atomicMax into colmax, which the caller zeroes).
cudaError_t launch_colmax(const float* yf, uint64_t rows_w, uint64_t rows_x, unsigned* colmax,
                          bool global, int num_sms, cudaStream_t s);
// quantize + pack of X' = yf^T with absmax `colmax` -> planes [n][rows_x][ceil(rows_w/32)],
// scales (rows_x or 1); flag[0] <- 1 on a non-finite absmax.
cudaError_t launch_requant_pack(const float* yf, uint64_t rows_w, uint64_t rows_x,
                                const unsigned* colmax, bool global, int n, uint32_t* planes,
                                double* scales, int* flag, cudaStream_t s);

// absmax bits (u32 of |float|) <-> doubles, for the split (multi-GPU) requant form
cudaError_t launch_bits_to_double(const unsigned* bits, uint64_t n, double* out, cudaStream_t s);
cudaError_t launch_double_to_bits(const double* in, uint64_t n, unsigned* bits, cudaStream_t s);

// recover (kernel.cpp:159-181) over a device plane-product stack [n_w*n_x][m*n] int32:
// y = sum 2^(i+j) stack[i][j] in int64, narrowed to int32. flags[0] <- 1 if an entry lies
// outside [-k, k] (PlaneProductStack ctor, kernel.cpp:91-101), flags[1] <- 1 if a recovered
// value does not fit int32 (kernel.cpp:172-176). Flags must be zero on entry.
cudaError_t launch_recover(const int32_t* stack, int n_w, int n_x, uint64_t mn, uint64_t k,
                           int32_t* y, int* flags, cudaStream_t s);

// ---- gemm_tc.cu ----------------------------------------------------------------------
struct GemmArgs {
  const uint8_t* codes_w;   // [rows_w x kpad]
  const uint8_t* codes_x;   // [rows_x x kpad]
  const int32_t* rowsum_w;  // [rows_w]
  const int32_t* rowsum_x;  // [round_up(rows_x, kRowsumPad)], zero padded
  uint64_t rows_w, rows_x, kpad, k_logical;
  int n_w, n_x;
  int32_t* y;               // int32 output [rows_w x rows_x] (or null)
  float* yf;                // dequant output (or null)
  const double* s_w;
  int gran_w;
  const double* s_x;
  int gran_x;
  int num_sms;
  unsigned long long* dbg = nullptr;  // optional wait-cycle counters (dev instrumentation)
  // dequant epilogue only: per-column (per-token) absmax of the f32 output as ordered u32
  // bits of |v| (atomicMax), or one global max when colmax_global; null = off
  unsigned* colmax = nullptr;
  bool colmax_global = false;
  unsigned long long* trace = nullptr;  // dev (APMM_TRACE): per-CTA globaltimer stamps [grid][8]
  bool early_w = true;  // PDL: the weight-plane GEMM may read W before the previous kernel ends
  // split-K weight-plane GEMM only: expand the feature planes and zero Y inside the kernel
  // (grid-wide barrier) instead of a K1x launch; null = K1x did it
  const uint32_t* xprep_planes = nullptr;
  uint64_t xprep_rows_pad = 0;
  unsigned long long* grid_bar = nullptr;
};
// Returns the number of kernel launches it enqueued via *launches.
cudaError_t launch_gemm_tc(const GemmArgs& a, cudaStream_t s, int* launches);
// ---- gemm_pair.cu (CTA-pair, 256x256 tiles) -------------------------------------------
// split_k: calls with too few 256x256 tiles: K split over the pairs, int32 partials TMA
// reduce-added into a Y the caller zeroed (K1 zero_out); int32 output, TMA-storable Y only.
cudaError_t launch_gemm_pair(const GemmArgs& a, cudaStream_t s, int* launches, bool split_k = false);

// ---- gemm_fused.cu (CTA pair, weight planes expanded on chip by transform warps) -------
// Needs the planes' row pitch (ceil(k/32) words) to be a multiple of 16 bytes and a 16-byte
// aligned base (TMA); a.codes_w is unused (K1 then runs with w_codes == nullptr and only
// produces rowsum_w).
bool gemm_fused_supported(const uint32_t* w_planes, uint64_t k);
bool gemm_wplanes_addressable(const uint32_t* w_planes, uint64_t k);
// split_k: mid-size calls (too few tiles for the machine): K split into units whose int32
// partials are TMA reduce-added into Y, which the caller must have zeroed (int32 out and
// TMA-storable Y only).
cudaError_t launch_gemm_pair_wplanes(const GemmArgs& a, const uint32_t* w_planes,
                                     cudaStream_t s, int* launches, bool split_k = false);

// ---- skinny.cu (few feature rows: weight planes streamed from HBM into mma.sync) -----
constexpr uint64_t kSkinnyMaxRowsX = 63;  // feature rows handled by K5 (+1 ones column <= 64)
constexpr uint64_t kSkinnyPreferRows = 40;  // above this the split-K K3f wins when it applies
struct SkinnyArgs {
  const uint32_t* w_planes;  // reference layout [n_w][rows_w][ceil(k/32)]
  const uint32_t* x_planes;  // reference layout [n_x][rows_x][ceil(k/32)]
  uint64_t rows_w, rows_x, k;
  int n_w, n_x;
  int32_t* y;
  float* yf;
  const double* s_w;
  int gran_w;
  const double* s_x;
  int gran_x;
  int num_sms;
  void* acc_ws;      // skinny_acc_bytes(): split-K accumulators, zero on entry, left zero
  void* scratch_ws;  // skinny_scratch_bytes(): feature fragments (2 halves) + weight repack
  int ws_half;       // ping-pong half for the feature fragments (PDL overlap of calls)
  bool early_w = true;  // PDL: stream weight planes before the previous kernel completes
  bool early_x = false;  // PDL: feature prep may read X before it (APMM_OPT_EARLY_FEATURE_READ)
  unsigned long long* trace = nullptr;  // dev (APMM_TRACE): per-CTA stamps [grid][8]
  // measurement (bench kernel pass): when non-null, recorded right before / after the
  // streaming kernel's launch (after the feature-prep kernel), with `ev_flags`
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
  unsigned ev_flags = 0;
};
size_t skinny_acc_bytes(uint64_t rows_w, uint64_t rows_x);
size_t skinny_scratch_bytes(uint64_t rows_w, uint64_t rows_x, uint64_t k, int n_w,
                            const void* w_planes);
cudaError_t launch_skinny(const SkinnyArgs& a, cudaStream_t s);
int skinny_launches(uint64_t rows_x);  // kernels launch_skinny issues (feature prep + K5, or K5)

// K6 (stream_tc.cu): weight planes streamed per warp, expanded in registers into TMEM (the
// MMA's A operand), features as u8 codes in shared memory (B), tcgen05 kind::i8, K split
// over every SM with int32 partials TMA reduce-added into a Y zeroed by the feature prep.
struct StreamTcArgs {
  const uint32_t* w_planes;  // reference layout [n_w][rows_w][ceil(k/32)]
  const uint32_t* x_planes;  // reference layout [n_x][rows_x][ceil(k/32)]
  uint64_t rows_w, rows_x, k;
  int n_w, n_x;
  int32_t* y;                // [rows_w][rows_x] int32
  int num_sms;
  void* ws;                  // stream_tc_ws_bytes(): feature codes + rowsum parts (+ padded Y)
  bool early_w = true;       // PDL: weight loads may start before the previous kernel completes
  bool early_x = false;      // PDL: the feature prep may read X before it
  unsigned long long* trace = nullptr;       // dev (APMM_TRACE): K6 per-CTA stamps [grid][8]
  unsigned long long* trace_prep = nullptr;  // dev (APMM_TRACE): prep per-block stamps
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;  // measurement: around the GEMM launch
  unsigned ev_flags = 0;
};
// Whether K6 can serve a call (shape, alignment and shared-memory budget).
bool stream_tc_supported(const uint32_t* w, uint64_t rows_w, uint64_t rows_x, uint64_t k, int n_w,
                         const void* y);
// Whether a call writes a padded Y in the workspace first (rows_x % 4 != 0 or Y not 16-byte
// aligned: the TMA reduce-adds need 16-byte rows) and copies it out.
bool stream_tc_padded(uint64_t rows_x, const void* y);
size_t stream_tc_ws_bytes(uint64_t rows_x, uint64_t k, uint64_t rows_w, bool padded);
cudaError_t launch_stream_tc(const StreamTcArgs& a, cudaStream_t s);

// Tensor-map encoder obtained from the driver through the runtime (no -lcuda).
// 2-D row-major tensor [outer x inner] with `stride_bytes` between rows, 128B swizzle.
CUresult encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dtype, uint32_t elem_bytes,
                        const void* base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                        uint32_t box_inner, uint32_t box_outer);
// 3-D u32 tensor, no swizzle, zero OOB fill: dims {inner, mid, outer}, byte strides of the
// mid and outer dimensions (multiples of 16).
CUresult encode_tmap_3d_u32(CUtensorMap* map, const void* base, const uint64_t (&dims)[3],
                            const uint64_t (&stride_bytes)[2], const uint32_t (&box)[3],
                            int swizzle_bytes = 0);  // 0: none, 32 / 64: SWIZZLE_32B / 64B

}  // namespace apmm_b200
