// prep.cu -- operand preparation kernels (HBM-bound, integer/byte work).
//
//   K1  expand          packed planes -> u8 codes for the tensor-core GEMM + rowsum(U)
//   K1' pack / unpack   decompose_and_pack / unpack (reference bitplane.cpp:48-84)
//   K2  quantize_pack   fp64 absmax quantize (bipolar.cpp:59-100) fused with the pack
//
// All kernels are bit-exact restatements of the reference semantics; the pack kernels
// build each 32-bit plane word with one warp ballot (lane k <-> column 32w+k), so a
// warp turns 32 codes into n plane words with n ballots and coalesced accesses.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "expand.cuh"
#include "internal.h"

namespace apmm_b200 {
namespace {

constexpr int kThreads = 256;

// ---- K1: planes -> u8 codes ------------------------------------------------------------
// Both GEMM operands in ONE launch (rows [0, rows_w) are W, the rest X), one warp per row,
// lanes striding over the 32-column words. A lane turns the n plane words of a 32-column
// group into 32 code bytes with an 8x8 bit transpose done SIMD across the 4 byte lanes of
// a 32-bit register (3 delta-swap stages, ~60 ALU ops for any n <= 8; rows i >= n are
// compile-time zero and fold away). The transpose leaves code(k = 8b + c) in byte b of
// output word c, i.e. the 32 codes of a group are stored in the K order
// (c, b) -> 4c + b instead of 8b + c. Both operands use the same order, and
// sum_k u_w(k) u_x(k) is invariant under a common permutation of k, so the GEMM result is
// unchanged; the zero padding lanes stay zero.
// rowsum(U) = sum_k u_k = sum_i 2^i popc(plane_i) comes straight from the planes.
constexpr int kExpandThreads = 128;  // small blocks: fit beside a resident GEMM CTA
using xpd::ExpandOperand;
using xpd::expand_one;
using xpd::transpose8;

// PDL protocol (see gemm_pair.cu). This kernel may start while the previous kernel in the
// stream (normally the previous call's GEMM) still runs. Before griddepcontrol.wait it
// touches only the WEIGHT planes (when early_w: weights are not produced by the kernel
// immediately before the call -- apmm_cuda.h, Conventions) and the workspace half that the
// GEMM two calls ago used (complete by construction). The feature planes -- possibly the
// previous kernel's output -- and the zeroing of Y are read / written only after the wait.
// It completes only after the previous kernel, so the next GEMM's wait on us covers both.
// NA / NB: the operands' plane counts at compile time (0: dispatched at run time, -1: the
// operand is absent). Single-operand launches (K1w weights, K1x features) use fixed counts.
template <int NA, int NB>
__device__ __forceinline__ void expand_sel(const ExpandOperand& op, uint32_t r, uint32_t wpr,
                                           uint32_t tail_mask, uint32_t kpad_words,
                                           uint32_t lane) {
  if constexpr (NA > 0) {
    xpd::expand_one_n<NA>(op, r, wpr, tail_mask, kpad_words, lane);
  } else {
    expand_one(op, r, wpr, tail_mask, kpad_words, lane);
  }
}

template <int NA, int NB>
__global__ void __launch_bounds__(kExpandThreads) expand_kernel(ExpandOperand a, ExpandOperand b,
                                                                 uint32_t wpr, uint32_t tail_mask,
                                                                 uint32_t kpad_words,
                                                                 uint4* zero_out, uint64_t zero_n,
                                                                 uint32_t early_w, uint32_t early_x,
                                                                 unsigned long long* ts) {
  // dev trace (APMM_TRACE): [0] start [1] W rows done [2] wait returned [3] end
  auto stamp = [&](int k) {
    if (ts && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ts[blockIdx.x * 8 + k] = t;
    }
  };
  stamp(0);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (!early_w) asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t warps = blockDim.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gwarp = blockIdx.x * warps + (threadIdx.x >> 5), nwarps = gridDim.x * warps;
  if constexpr (NA >= 0) {
    for (uint32_t r = gwarp; r < a.rows; r += nwarps) {
      expand_sel<NA, 0>(a, r, wpr, tail_mask, kpad_words, lane);
    }
  }
  // X rows continue the W rows' round robin, so a grid-stride pass over both stays balanced
  const uint32_t xr0 = NA >= 0 ? (gwarp + nwarps - a.rows % nwarps) % nwarps : gwarp;
  if constexpr (NB >= 0) {
    if (early_x) {
      for (uint32_t r = xr0; r < b.rows; r += nwarps) {
        expand_sel<NB, 0>(b, r, wpr, tail_mask, kpad_words, lane);
      }
    }
  }
  if (blockIdx.x == 0) {
    for (uint32_t r = a.rows + threadIdx.x; r < a.rows_pad; r += blockDim.x) a.rowsum[r] = 0;
    for (uint32_t r = b.rows + threadIdx.x; r < b.rows_pad; r += blockDim.x) b.rowsum[r] = 0;
  }
  stamp(1);
  if (early_w) asm volatile("griddepcontrol.wait;" ::: "memory");
  stamp(2);
  if constexpr (NB >= 0) {
    if (!early_x) {
      for (uint32_t r = xr0; r < b.rows; r += nwarps) {
        expand_sel<NB, 0>(b, r, wpr, tail_mask, kpad_words, lane);
      }
    }
  }
  // split-K GEMMs reduce-add into Y: zero it here, after the previous kernel in the stream
  // (which may still have been writing the same Y) has completed
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < zero_n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    zero_out[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  stamp(3);
}

// ---- K1': codes -> planes (decompose_and_pack) -------------------------------------------
// One warp per (row, word). Lane k holds code (r, 32w+k); plane word i = ballot(bit i).
__global__ void __launch_bounds__(kThreads) pack_kernel(const uint8_t* __restrict__ codes,
                                                         uint64_t rows, uint64_t cols, int n,
                                                         uint32_t* __restrict__ planes) {
  const uint64_t wpr = (cols + 31) / 32;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (gw >= rows * wpr) return;  // warp-uniform
  const uint64_t r = gw / wpr, w = gw % wpr;
  const uint64_t col = w * 32 + lane;
  const uint32_t c = col < cols ? codes[r * cols + col] : 0u;
  uint32_t mine = 0;
  for (int i = 0; i < n; ++i) {
    const uint32_t word = __ballot_sync(0xffffffffu, (c >> i) & 1u);
    if (int(lane) == i) mine = word;
  }
  if (int(lane) < n) planes[(uint64_t(lane) * rows + r) * wpr + w] = mine;
}

// ---- unpack ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) unpack_kernel(const uint32_t* __restrict__ planes,
                                                           uint64_t rows, uint64_t cols, int n,
                                                           uint8_t* __restrict__ codes) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const uint64_t wpr = (cols + 31) / 32;
  const uint64_t r = e / cols, k = e % cols;
  uint32_t c = 0;
  for (int i = 0; i < n; ++i) {
    c |= ((__ldg(planes + (uint64_t(i) * rows + r) * wpr + (k >> 5)) >> (k & 31)) & 1u) << i;
  }
  codes[e] = static_cast<uint8_t>(c);
}

// ---- K2: fp64 quantize + pack ----------------------------------------------------------------
// round_to_grid (bipolar.cpp:63-68) with explicitly rounded IEEE ops so no FMA contraction
// can change a result relative to the reference's x86 SSE2 arithmetic.
__device__ __forceinline__ uint32_t quantize_code(double x, double s, int maxv) {
  const double t = __ddiv_rn(x, s);
  const double q = __dadd_rn(__dmul_rn(2.0, floor(__ddiv_rn(t, 2.0))), 1.0);
  int qi;
  if (q > double(maxv)) qi = maxv;
  else if (q < -double(maxv)) qi = -maxv;
  else qi = static_cast<int>(q);
  return static_cast<uint32_t>((qi + maxv) / 2);
}

// Same result as quantize_code without the fp64 division and without fp64 conversions
// (cvt runs on a slow pipe) on almost every element. The code depends on x / s only through
// h = floor(RN(x/s) / 2) = floor(RN(x / (2s))) (halving is exact). With r2 = RN(1 / (2s)),
// u = RN(x * r2) is within ~2 ulps of RN(x / (2s)), |u| <= 2^8 for every admissible code, so
// |u - RN(x/(2s))| < 2^-43. floor(u) comes from the 1.5 * 2^52 rounding trick (two DADDs,
// integer bits). If u lies farther than 2^-40 from an integer, floor(u) is the reference's
// floor; otherwise (values on a grid boundary, subnormal quotients) the exact division
// decides. Zero maps to q = 1 directly (x / s = +-0).
// r2 = RN(1 / (2s)) for the fast paths, or 0 (u = 0 lands in the guard band, so every element
// takes the exact division) when it would not be a normal double with margin
__device__ __forceinline__ double fast_recip(double s) {
  const double r2 = __ddiv_rn(1.0, __dmul_rn(2.0, s));
  return (r2 >= 0x1p-1000 && r2 <= 0x1p1000) ? r2 : 0.0;
}
__device__ __forceinline__ uint32_t code_of_q(int q, int maxv) {
  q = q > maxv ? maxv : (q < -maxv ? -maxv : q);
  return static_cast<uint32_t>((q + maxv) / 2);
}
__device__ __forceinline__ uint32_t quantize_code_fast(double x, double s, double r2, int maxv) {
  if (x == 0.0) return static_cast<uint32_t>((1 + maxv) / 2);
  const double u = __dmul_rn(x, r2);
  if (fabs(u) < 0x1p40) {
    const double t = __dadd_rn(u, 6755399441055744.0);  // 1.5 * 2^52: RN(u) in the low bits
    const double back = __dsub_rn(t, 6755399441055744.0);
    int n = __double2loint(t);
    const bool above = back > u;
    const double frac = __dsub_rn(u, above ? __dsub_rn(back, 1.0) : back);
    if (frac > 0x1p-40 && frac < 1.0 - 0x1p-40) return code_of_q(2 * (n - (above ? 1 : 0)) + 1, maxv);
  }
  return quantize_code(x, s, maxv);
}
// f32 input (the dequantized GEMM output): the approximation in FP32 (error < 2^-15 for
// |u| <= 2^8) with a 2^-14 guard band, the exact fp64 path otherwise.
__device__ __forceinline__ uint32_t quantize_code_f32(float v, double s, float r2f, int maxv) {
  if (v == 0.0f) return static_cast<uint32_t>((1 + maxv) / 2);
  const float u = __fmul_rn(v, r2f);
  if (fabsf(u) < 4194304.0f) {
    const float t = __fadd_rn(u, 12582912.0f);  // 1.5 * 2^23: RN(u) in the low bits
    const float back = __fsub_rn(t, 12582912.0f);
    const int n = __float_as_int(t) - 0x4B400000;
    const bool above = back > u;
    const float frac = __fsub_rn(u, above ? __fsub_rn(back, 1.0f) : back);
    if (frac > 0x1p-14f && frac < 1.0f - 0x1p-14f) return code_of_q(2 * (n - (above ? 1 : 0)) + 1, maxv);
  }
  return quantize_code(static_cast<double>(v), s, maxv);
}

// Optional GEMM-operand output (K2 feeding K3 without planes): `codes` = u8 codes
// [rows][kpad] in K1's permuted order (column 8b + c of each 32-column group at byte 4c + b).
struct GemmCodesOut {
  uint8_t* codes;   // null: no GEMM-layout output
  int32_t* rowsum;  // [rows_pad], zeroed by the launcher
  uint64_t kpad;
};

// Returns the lane's code (0 past the row end) so callers can form rowsum(U).
__device__ __forceinline__ uint32_t quantize_pack_word(const double* __restrict__ xrow,
                                                       uint64_t r, uint64_t rows, uint64_t cols,
                                                       uint64_t w, int n, int maxv, double s,
                                                       double r2, uint32_t* __restrict__ planes,
                                                       uint8_t* __restrict__ codes,
                                                       const GemmCodesOut& g) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t wpr = (cols + 31) / 32;
  const uint64_t col = w * 32 + lane;
  uint32_t c = 0;
  if (col < cols) {
    c = quantize_code_fast(xrow[col], s, r2, maxv);
    if (codes) codes[r * cols + col] = static_cast<uint8_t>(c);
  }
  if (g.codes) {
    g.codes[r * g.kpad + w * 32 + (lane & 7u) * 4 + (lane >> 3)] = static_cast<uint8_t>(c);
  }
  if (planes) {
    uint32_t mine = 0;
    for (int i = 0; i < n; ++i) {
      const uint32_t word = __ballot_sync(0xffffffffu, (c >> i) & 1u);
      if (int(lane) == i) mine = word;
    }
    if (int(lane) < n) planes[(uint64_t(lane) * rows + r) * wpr + w] = mine;
  }
  return c;
}

// zero K padding of the GEMM-layout codes: bytes [32 * wpr, kpad) of row r, one warp
__device__ __forceinline__ void zero_code_tail(const GemmCodesOut& g, uint64_t r, uint64_t cols) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t b = ((cols + 31) / 32) * 32 + lane; b < g.kpad; b += 32) g.codes[r * g.kpad + b] = 0;
}

// Per-row granularity: one block per row (absmax reduce, then quantize+pack its words).
__global__ void __launch_bounds__(kThreads)
    quantize_rows_kernel(const double* __restrict__ x, uint64_t rows, uint64_t cols, int n,
                         uint32_t* __restrict__ planes, double* __restrict__ scales,
                         uint8_t* __restrict__ codes, int* __restrict__ flag,
                         GemmCodesOut g) {
  const uint64_t r = blockIdx.x;
  const double* xrow = x + r * cols;
  const int maxv = (1 << n) - 1;
  double amax = 0.0;
  int bad = 0;
  for (uint64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    const double v = xrow[c];
    if (!isfinite(v)) bad = 1;
    amax = fmax(amax, fabs(v));
  }
  __shared__ double red[kThreads / 32];
  __shared__ int redbad;
  if (threadIdx.x == 0) redbad = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  __syncthreads();
  if (bad) atomicOr(&redbad, 1);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
  __syncthreads();
  double m = 0.0;
  for (int i = 0; i < int(blockDim.x / 32); ++i) m = fmax(m, red[i]);
  if (redbad) {
    if (threadIdx.x == 0) atomicOr(flag, 1);
    return;
  }
  const double s = m == 0.0 ? 1.0 : __ddiv_rn(m, double(maxv));  // bipolar.cpp:91
  const double r2 = fast_recip(s);  // quantize_code_fast
  if (threadIdx.x == 0) scales[r] = s;
  const uint64_t wpr = (cols + 31) / 32;
  int32_t rsum = 0;
  for (uint64_t w = threadIdx.x >> 5; w < wpr; w += blockDim.x / 32) {
    rsum += static_cast<int32_t>(quantize_pack_word(xrow, r, rows, cols, w, n, maxv, s, r2, planes,
                                                    codes, g));
  }
  if (g.codes) {
    if (threadIdx.x < 32) zero_code_tail(g, r, cols);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
    __shared__ int32_t rred[kThreads / 32];
    if ((threadIdx.x & 31) == 0) rred[threadIdx.x >> 5] = rsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      int32_t t = 0;
      for (int i = 0; i < int(blockDim.x / 32); ++i) t += rred[i];
      g.rowsum[r] = t;
    }
  }
}

// Per-tensor granularity, pass 1: global absmax (non-negative doubles order like their
// u64 bit patterns, so atomicMax on the bits is exact) + non-finite flag.
__global__ void __launch_bounds__(kThreads) absmax_kernel(const double* __restrict__ x,
                                                           uint64_t count,
                                                           unsigned long long* amax_bits,
                                                           int* flag) {
  double amax = 0.0;
  int bad = 0;
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const double v = x[e];
    if (!isfinite(v)) bad = 1;
    amax = fmax(amax, fabs(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(amax_bits, static_cast<unsigned long long>(__double_as_longlong(amax)));
    if (bad) atomicOr(flag, 1);
  }
}

// Per-tensor pass 2: warp per (row, word).
__global__ void __launch_bounds__(kThreads)
    quantize_tensor_kernel(const double* __restrict__ x, uint64_t rows, uint64_t cols, int n,
                           const unsigned long long* amax_bits, uint32_t* __restrict__ planes,
                           double* __restrict__ scales, uint8_t* __restrict__ codes,
                           const int* flag, GemmCodesOut g) {
  if (*flag) return;
  const int maxv = (1 << n) - 1;
  const double m = __longlong_as_double(static_cast<long long>(*amax_bits));
  const double s = m == 0.0 ? 1.0 : __ddiv_rn(m, double(maxv));
  const double r2 = fast_recip(s);  // quantize_code_fast
  if (blockIdx.x == 0 && threadIdx.x == 0) scales[0] = s;
  const uint64_t wpr = (cols + 31) / 32;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (gw >= rows * wpr) return;
  const uint64_t r = gw / wpr, w = gw % wpr;
  int32_t c = static_cast<int32_t>(
      quantize_pack_word(x + r * cols, r, rows, cols, w, n, maxv, s, r2, planes, codes, g));
  if (g.codes) {  // one atomic per (row, word) into the zeroed rowsum
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(g.rowsum + r, c);
    if (w == wpr - 1) zero_code_tail(g, r, cols);
  }
}

// recover: one thread per output element, int64 accumulation of the shifted plane products
__global__ void __launch_bounds__(kThreads) recover_kernel(const int32_t* __restrict__ stack,
                                                           int n_w, int n_x, uint64_t mn,
                                                           int64_t k, int32_t* __restrict__ y,
                                                           int* __restrict__ flags) {
  const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= mn) return;
  int64_t acc = 0;
  bool range_ok = true;
  for (int i = 0; i < n_w; ++i) {
    for (int j = 0; j < n_x; ++j) {
      const int64_t v = __ldg(stack + uint64_t(i * n_x + j) * mn + e);
      range_ok &= v <= k && v >= -k;
      acc += v * (int64_t(1) << (i + j));
    }
  }
  if (!range_ok) atomicOr(flags + 0, 1);
  if (acc > INT32_MAX || acc < INT32_MIN) atomicOr(flags + 1, 1);
  y[e] = static_cast<int32_t>(acc);
}

// ---- dot_1bit_xor (kernel.cpp:115-123): k - 2 popc(a ^ b), one block -----------------
__global__ void __launch_bounds__(kThreads) dot_xor_kernel(const uint32_t* __restrict__ a,
                                                            const uint32_t* __restrict__ b,
                                                            uint64_t words, uint64_t k,
                                                            int64_t* out) {
  uint64_t pc = 0;
  for (uint64_t w = threadIdx.x; w < words; w += blockDim.x) pc += __popc(__ldg(a + w) ^ __ldg(b + w));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, o);
  __shared__ uint64_t part[kThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = pc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int i = 0; i < kThreads / 32; ++i) t += part[i];
    *out = static_cast<int64_t>(k) - 2 * static_cast<int64_t>(t);
  }
}

// ---- to_real (tensor_file.cpp:115-120): f32 payload -> f64 values -------------------------
__global__ void __launch_bounds__(kThreads) widen_kernel(const float* __restrict__ src,
                                                          uint64_t n, double* __restrict__ dst) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += uint64_t(gridDim.x) * blockDim.x) {
    dst[e] = static_cast<double>(src[e]);
  }
}

// ---- next-layer requantization -------------------------------------
// yf: the dequantized GEMM output [rows_w][rows_x] f32 (rows = output features, columns =
// tokens); the next layer's activation is X' = yf^T [rows_x tokens][rows_w features].
// Column absmax when the GEMM epilogue did not form it (skinny / weight-plane routes):
// thread per column over a slab of rows, one atomicMax per (thread, slab).
__global__ void __launch_bounds__(kThreads) colmax_kernel(const float* __restrict__ yf,
                                                           uint64_t rows_w, uint64_t rows_x,
                                                           uint64_t rows_per_slab,
                                                           unsigned* colmax, int global) {
  const uint64_t c = uint64_t(blockIdx.x) * 32 + (threadIdx.x & 31);
  const uint64_t r0 = uint64_t(blockIdx.y) * rows_per_slab;
  const uint64_t r1 = r0 + rows_per_slab < rows_w ? r0 + rows_per_slab : rows_w;
  uint32_t m = 0;
  if (c < rows_x) {
    const uint64_t step = blockDim.x / 32;
    uint64_t r = r0 + (threadIdx.x >> 5);
    for (; r + 7 * step < r1; r += 8 * step) {  // 8 loads in flight per thread
      uint32_t b[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) b[u] = __float_as_uint(__ldg(yf + (r + u * step) * rows_x + c));
#pragma unroll
      for (int u = 0; u < 8; ++u) m = (b[u] & 0x7fffffffu) > m ? (b[u] & 0x7fffffffu) : m;
    }
    for (; r < r1; r += step) {
      const uint32_t b = __float_as_uint(__ldg(yf + r * rows_x + c)) & 0x7fffffffu;
      m = b > m ? b : m;
    }
  }
  if (global) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint32_t t = __shfl_xor_sync(0xffffffffu, m, o);
      m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(colmax, m);
  } else if (c < rows_x) {
    atomicMax(colmax + c, m);
  }
}

// quantize (bipolar.cpp:72-100) of X' with the reduced absmax, then decompose_and_pack
// (bitplane.cpp:48-66): block = 8 warps x (32 tokens, 8 consecutive plane words). Warp q
// reads yf rows 32(w0+q) .. +31 for 32 tokens (coalesced 128-B rows), lane = token, and
// builds its token's n plane words bit by bit; the words go through shared memory so each
// (plane, token) row receives 8 consecutive words (32-B sectors) per block.
__global__ void bits_to_double_kernel(const unsigned* bits, uint64_t n, double* out) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    out[i] = static_cast<double>(__uint_as_float(bits[i]));
  }
}
// inverse (absmax values of the f32 output, exactly representable as float); a non-finite
// value maps to the inf/NaN bit patterns so the pack kernel reports it
__global__ void double_to_bits_kernel(const double* in, uint64_t n, unsigned* bits) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    bits[i] = __float_as_uint(fabsf(static_cast<float>(in[i])));
  }
}

constexpr int kRqWords = 8;
template <int N>
__global__ void __launch_bounds__(kThreads) requant_pack_kernel(
    const float* __restrict__ yf, uint64_t rows_w, uint64_t rows_x, const unsigned* colmax,
    int global, uint32_t* __restrict__ planes, double* __restrict__ scales, int* flag) {
  constexpr int n = N;  // planes of the next layer's activation (compile time: the bit
                        // inserts below run for live planes only)
  __shared__ uint32_t sw[8][32][kRqWords + 1];
  const uint32_t lane = threadIdx.x & 31, q = threadIdx.x >> 5;
  const uint64_t wpr = (rows_w + 31) / 32;
  // blockIdx.x = token block (fastest): the resident blocks read whole rows of yf (all
  // tokens) at once, so DRAM pages are used fully (word groups first read 128 B per row)
  const uint64_t t = uint64_t(blockIdx.x) * 32 + lane;
  const uint64_t w = uint64_t(blockIdx.y) * kRqWords + q;
  const int maxv = (1 << n) - 1;
  const uint32_t mbits = global ? colmax[0] : (t < rows_x ? colmax[t] : 0u);
  const double m = static_cast<double>(__uint_as_float(mbits));
  const bool finite = mbits < 0x7f800000u;
  if (!finite && t < rows_x) atomicOr(flag, 1);
  const double s = m == 0.0 ? 1.0 : __ddiv_rn(m, double(maxv));  // bipolar.cpp:91
  const double r2 = fast_recip(s);
  // fast FP32 path only where RN(1/(2s)) is a normal float with margin (else r2f = 0: every
  // element takes the exact path, see quantize_code_f32)
  const float r2f = (r2 >= 0x1p-120 && r2 <= 0x1p120) ? static_cast<float>(r2) : 0.0f;
  if (blockIdx.y == 0 && q == 0 && finite) {
    if (global) {
      if (blockIdx.x == 0 && lane == 0) scales[0] = s;
    } else if (t < rows_x) {
      scales[t] = s;
    }
  }
  uint32_t word[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (t < rows_x && w < wpr && finite) {
    const uint64_t r0 = w * 32;
    const uint32_t nr = rows_w - r0 < 32 ? static_cast<uint32_t>(rows_w - r0) : 32u;
    // all 32 loads first (one memory round trip per thread, not 32 dependent ones)
    float v[32];
#pragma unroll
    for (uint32_t j = 0; j < 32; ++j) v[j] = j < nr ? __ldg(yf + (r0 + j) * rows_x + t) : 0.0f;
#pragma unroll
    for (uint32_t j = 0; j < 32; ++j) {
      const uint32_t c = j < nr ? quantize_code_f32(v[j], s, r2f, maxv) : 0u;
#pragma unroll
      for (int i = 0; i < N; ++i) word[i] |= ((c >> i) & 1u) << j;
    }
  }
#pragma unroll
  for (int i = 0; i < N; ++i) sw[i][lane][q] = word[i];
  __syncthreads();
  // write out: thread = (plane i, token, word) with the word index fastest
  const uint64_t w0 = uint64_t(blockIdx.y) * kRqWords;
  for (uint32_t e = threadIdx.x; e < uint32_t(n) * 32u * kRqWords; e += blockDim.x) {
    const uint32_t qq = e % kRqWords, tok = (e / kRqWords) % 32, i = e / (kRqWords * 32);
    const uint64_t tt = uint64_t(blockIdx.x) * 32 + tok, ww = w0 + qq;
    if (tt < rows_x && ww < wpr) planes[(uint64_t(i) * rows_x + tt) * wpr + ww] = sw[i][tok][qq];
  }
}

unsigned blocks_for(uint64_t threads) {
  return static_cast<unsigned>((threads + kThreads - 1) / kThreads);
}

}  // namespace

cudaError_t launch_expand(const uint32_t* w_planes, uint64_t rows_w, int n_w,
                          uint8_t* w_codes, int32_t* w_rowsum, const uint32_t* x_planes,
                          uint64_t rows_x, uint64_t rows_x_pad, int n_x, uint8_t* x_codes,
                          int32_t* x_rowsum, uint64_t cols, uint64_t kpad, int num_sms,
                          cudaStream_t s, void* zero_out, uint64_t zero_bytes, bool early_w,
                          bool early_x, unsigned long long* trace, int blocks_per_sm) {
  const uint32_t wpr = static_cast<uint32_t>((cols + 31) / 32);
  const uint32_t tail = static_cast<uint32_t>(cols & 31);
  const uint32_t tail_mask = tail ? ((1u << tail) - 1u) : 0xffffffffu;
  // Weight codes are written while the previous GEMM runs (PDL) and are far larger than its
  // L2 working set at large shapes (70B FFN: 235 MB): streaming stores keep them from
  // evicting the running GEMM's operand tiles. APMM_K1_CS (dev builds) overrides: bit 0 =
  // weights, bit 1 = features.
  static const int cs_env = [] {
    const char* e = APMM_DEV_ENV("APMM_K1_CS");
    return e ? std::atoi(e) : -1;
  }();
  const int cs_w = cs_env >= 0 ? (cs_env & 1) : 1, cs_x = cs_env >= 0 ? ((cs_env >> 1) & 1) : 0;
  const ExpandOperand a{w_planes, w_codes, w_rowsum, static_cast<uint32_t>(rows_w),
                        static_cast<uint32_t>(rows_w), n_w, cs_w};
  const ExpandOperand b{x_planes, x_codes, x_rowsum, static_cast<uint32_t>(rows_x),
                        static_cast<uint32_t>(rows_x_pad), n_x, cs_x};
  const uint64_t warps_needed = rows_w + rows_x;
  uint64_t blocks = (warps_needed + kExpandThreads / 32 - 1) / (kExpandThreads / 32);
  if (zero_bytes && blocks < uint64_t(num_sms)) blocks = num_sms;  // the zeroing is grid-wide
  // one block per SM when the launch overlaps a running GEMM (early reads): every block fits
  // beside the resident GEMM CTA (regs: 8 x 192 x 32 + 4 x 80 x 32 <= 64K), so none is left
  // waiting behind blocks parked in griddepcontrol.wait. A launch that only works after the
  // previous kernel completed (blocks_per_sm > 1) has the whole machine: more warps, more
  // loads in flight (the expansion is latency bound at one 4-warp block per SM).
  const uint64_t cap = uint64_t(num_sms) * uint64_t(blocks_per_sm < 1 ? 1 : blocks_per_sm);
  if (blocks > cap) blocks = cap;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(kExpandThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // single-operand launches (one side has no rows) get a kernel specialised on its plane
  // count; the combined launch dispatches per row at run time
  const uint32_t kw = static_cast<uint32_t>(kpad / 32);
  uint4* zo = static_cast<uint4*>(zero_out);
  const uint64_t zn = zero_bytes / 16;
  const uint32_t ew = early_w ? 1u : 0u, ex = early_x ? 1u : 0u;
  cudaError_t e;
#define APMM_K1_ONE(KA, KB) \
  cudaLaunchKernelEx(&cfg, expand_kernel<KA, KB>, a, b, wpr, tail_mask, kw, zo, zn, ew, ex, trace)
  // (the absent side keeps its rowsum padding zeroing, done by block 0 for both operands)
  if (rows_x == 0 && w_codes != nullptr && n_w >= 1 && n_w <= 8) {
    switch (n_w) {
      case 1: e = APMM_K1_ONE(1, -1); break;
      case 2: e = APMM_K1_ONE(2, -1); break;
      case 3: e = APMM_K1_ONE(3, -1); break;
      case 4: e = APMM_K1_ONE(4, -1); break;
      case 5: e = APMM_K1_ONE(5, -1); break;
      case 6: e = APMM_K1_ONE(6, -1); break;
      case 7: e = APMM_K1_ONE(7, -1); break;
      default: e = APMM_K1_ONE(8, -1); break;
    }
  } else if (rows_w == 0 && n_x >= 1 && n_x <= 8) {
    switch (n_x) {
      case 1: e = APMM_K1_ONE(-1, 1); break;
      case 2: e = APMM_K1_ONE(-1, 2); break;
      case 3: e = APMM_K1_ONE(-1, 3); break;
      case 4: e = APMM_K1_ONE(-1, 4); break;
      case 5: e = APMM_K1_ONE(-1, 5); break;
      case 6: e = APMM_K1_ONE(-1, 6); break;
      case 7: e = APMM_K1_ONE(-1, 7); break;
      default: e = APMM_K1_ONE(-1, 8); break;
    }
  } else {
    e = APMM_K1_ONE(0, 0);
  }
#undef APMM_K1_ONE
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_recover(const int32_t* stack, int n_w, int n_x, uint64_t mn, uint64_t k,
                           int32_t* y, int* flags, cudaStream_t s) {
  if (mn == 0) return cudaSuccess;
  recover_kernel<<<blocks_for(mn), kThreads, 0, s>>>(stack, n_w, n_x, mn, static_cast<int64_t>(k),
                                                     y, flags);
  return cudaGetLastError();
}

cudaError_t launch_pack(const uint8_t* codes, uint64_t rows, uint64_t cols, int n,
                        uint32_t* planes, cudaStream_t s) {
  const uint64_t warps = rows * ((cols + 31) / 32);
  pack_kernel<<<blocks_for(warps * 32), kThreads, 0, s>>>(codes, rows, cols, n, planes);
  return cudaGetLastError();
}

cudaError_t launch_unpack(const uint32_t* planes, uint64_t rows, uint64_t cols, int n,
                          uint8_t* codes, cudaStream_t s) {
  unpack_kernel<<<blocks_for(rows * cols), kThreads, 0, s>>>(planes, rows, cols, n, codes);
  return cudaGetLastError();
}

cudaError_t launch_quantize_pack(const double* x, uint64_t rows, uint64_t cols, int n,
                                 int granularity, uint32_t* planes, double* scales,
                                 uint8_t* codes, unsigned long long* amax_bits, int* flag,
                                 cudaStream_t s, uint8_t* gemm_codes, int32_t* gemm_rowsum,
                                 uint64_t kpad, uint64_t rowsum_pad) {
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  const GemmCodesOut g{gemm_codes, gemm_rowsum, kpad};
  if (gemm_codes) {  // rowsum: zero the padding (and, per tensor, the atomics' targets)
    e = cudaMemsetAsync(gemm_rowsum, 0, rowsum_pad * sizeof(int32_t), s);
    if (e != cudaSuccess) return e;
  }
  if (granularity == 1) {
    quantize_rows_kernel<<<static_cast<unsigned>(rows), kThreads, 0, s>>>(x, rows, cols, n,
                                                                          planes, scales, codes,
                                                                          flag, g);
    return cudaGetLastError();
  }
  e = cudaMemsetAsync(amax_bits, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  const uint64_t count = rows * cols;
  unsigned grid = blocks_for(count);
  if (grid > 148u * 8u) grid = 148u * 8u;
  absmax_kernel<<<grid, kThreads, 0, s>>>(x, count, amax_bits, flag);
  const uint64_t warps = rows * ((cols + 31) / 32);
  quantize_tensor_kernel<<<blocks_for(warps * 32), kThreads, 0, s>>>(x, rows, cols, n, amax_bits,
                                                                     planes, scales, codes, flag, g);
  return cudaGetLastError();
}

// ---- tensor maps ------------------------------------------------------------------------------
namespace {
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr) {
      return nullptr;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return encode;
}
}  // namespace

CUresult encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dtype, uint32_t /*elem_bytes*/,
                        const void* base, uint64_t inner, uint64_t outer, uint64_t stride_bytes,
                        uint32_t box_inner, uint32_t box_outer) {
  auto encode = tmap_encoder();
  if (!encode) return CUDA_ERROR_NOT_FOUND;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {stride_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t elem_strides[2] = {1, 1};
  return encode(map, dtype, 2, const_cast<void*>(base), dims, strides, box, elem_strides,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

CUresult encode_tmap_3d_u32(CUtensorMap* map, const void* base, const uint64_t (&dims)[3],
                            const uint64_t (&stride_bytes)[2], const uint32_t (&box)[3],
                            int swizzle_bytes) {
  auto encode = tmap_encoder();
  if (!encode) return CUDA_ERROR_NOT_FOUND;
  const cuuint64_t d[3] = {dims[0], dims[1], dims[2]};
  const cuuint64_t st[2] = {stride_bytes[0], stride_bytes[1]};
  const cuuint32_t b[3] = {box[0], box[1], box[2]};
  const cuuint32_t es[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(base), d, st, b, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE,
                swizzle_bytes == 64   ? CU_TENSOR_MAP_SWIZZLE_64B
                : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                      : CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

cudaError_t launch_dot_xor(const uint32_t* a, const uint32_t* b, uint64_t words, uint64_t k,
                           int64_t* out, cudaStream_t s) {
  dot_xor_kernel<<<1, kThreads, 0, s>>>(a, b, words, k, out);
  return cudaGetLastError();
}

cudaError_t launch_widen(const float* src, uint64_t n, double* dst, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t blocks = (n + kThreads - 1) / kThreads;
  if (blocks > 4096) blocks = 4096;
  widen_kernel<<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(src, n, dst);
  return cudaGetLastError();
}

cudaError_t launch_colmax(const float* yf, uint64_t rows_w, uint64_t rows_x, unsigned* colmax,
                          bool global, int num_sms, cudaStream_t s) {
  const uint64_t cblocks = (rows_x + 31) / 32;
  uint64_t slabs = (uint64_t(4) * num_sms + cblocks - 1) / cblocks;
  const uint64_t max_slabs = (rows_w + 63) / 64;
  if (slabs > max_slabs) slabs = max_slabs;
  if (slabs < 1) slabs = 1;
  if (slabs > 65535) slabs = 65535;
  const uint64_t per = (rows_w + slabs - 1) / slabs;
  colmax_kernel<<<dim3(static_cast<unsigned>(cblocks), static_cast<unsigned>(slabs)), kThreads, 0,
                  s>>>(yf, rows_w, rows_x, per, colmax, global ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_bits_to_double(const unsigned* bits, uint64_t n, double* out, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>(n / kThreads + 1 < 1024 ? n / kThreads + 1 : 1024);
  bits_to_double_kernel<<<blocks, kThreads, 0, s>>>(bits, n, out);
  return cudaGetLastError();
}

cudaError_t launch_double_to_bits(const double* in, uint64_t n, unsigned* bits, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>(n / kThreads + 1 < 1024 ? n / kThreads + 1 : 1024);
  double_to_bits_kernel<<<blocks, kThreads, 0, s>>>(in, n, bits);
  return cudaGetLastError();
}

cudaError_t launch_requant_pack(const float* yf, uint64_t rows_w, uint64_t rows_x,
                                const unsigned* colmax, bool global, int n, uint32_t* planes,
                                double* scales, int* flag, cudaStream_t s) {
  const uint64_t wpr = (rows_w + 31) / 32;
  const dim3 grid(static_cast<unsigned>((rows_x + 31) / 32),
                  static_cast<unsigned>((wpr + kRqWords - 1) / kRqWords));
  switch (n) {
#define APMM_RQ(NN) \
  case NN: \
    requant_pack_kernel<NN><<<grid, kThreads, 0, s>>>(yf, rows_w, rows_x, colmax, global ? 1 : 0, \
                                                      planes, scales, flag); \
    break;
    APMM_RQ(1) APMM_RQ(2) APMM_RQ(3) APMM_RQ(4) APMM_RQ(5) APMM_RQ(6) APMM_RQ(7) APMM_RQ(8)
#undef APMM_RQ
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace apmm_b200
