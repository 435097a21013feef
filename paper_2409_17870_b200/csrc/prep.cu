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

#include "internal.h"

namespace apmm_b200 {
namespace {

constexpr int kThreads = 256;

// Spread a 4-bit nibble x into bit 0 of four bytes: (x*0x00204081) places bit b at
// 7b+b = 8b with no carries (partial products occupy disjoint bit ranges).
__device__ __forceinline__ uint32_t spread4(uint32_t x) { return (x * 0x00204081u) & 0x01010101u; }

// ---- K1: planes -> u8 codes ------------------------------------------------------------
// One block per row. Thread handles 32-column words w; each word yields 32 code bytes.
// rowsum(U) = sum_k u_k = sum_i 2^i popc(plane_i) -- computed from the planes directly.
__global__ void __launch_bounds__(kThreads) expand_kernel(const uint32_t* __restrict__ planes,
                                                           uint32_t rows, uint32_t wpr, int n,
                                                           uint32_t tail_mask,
                                                           uint8_t* __restrict__ codes,
                                                           uint32_t kpad_words,
                                                           int32_t* __restrict__ rowsum) {
  const uint32_t r = blockIdx.x;
  int32_t sum = 0;
  uint8_t* dst_row = codes + uint64_t(r) * kpad_words * 32u;
  for (uint32_t w = threadIdx.x; w < kpad_words; w += blockDim.x) {
    uint32_t out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (w < wpr) {
      for (int i = 0; i < n; ++i) {
        uint32_t b = __ldg(planes + (uint64_t(i) * rows + r) * wpr + w);
        if (w == wpr - 1) b &= tail_mask;  // padding lanes are zero by contract; enforce it
        sum += __popc(b) << i;
#pragma unroll
        for (int j = 0; j < 8; ++j) out[j] |= spread4((b >> (4 * j)) & 0xFu) << i;
      }
    }
    uint4* d = reinterpret_cast<uint4*>(dst_row + uint64_t(w) * 32u);
    d[0] = make_uint4(out[0], out[1], out[2], out[3]);
    d[1] = make_uint4(out[4], out[5], out[6], out[7]);
  }
  // block reduction of the row sum
  __shared__ int32_t red[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t s = 0;
    for (int i = 0; i < int(blockDim.x / 32); ++i) s += red[i];
    rowsum[r] = s;
  }
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

__device__ __forceinline__ void quantize_pack_word(const double* __restrict__ xrow,
                                                   uint64_t r, uint64_t rows, uint64_t cols,
                                                   uint64_t w, int n, int maxv, double s,
                                                   uint32_t* __restrict__ planes,
                                                   uint8_t* __restrict__ codes) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t wpr = (cols + 31) / 32;
  const uint64_t col = w * 32 + lane;
  uint32_t c = 0;
  if (col < cols) {
    c = quantize_code(xrow[col], s, maxv);
    if (codes) codes[r * cols + col] = static_cast<uint8_t>(c);
  }
  uint32_t mine = 0;
  for (int i = 0; i < n; ++i) {
    const uint32_t word = __ballot_sync(0xffffffffu, (c >> i) & 1u);
    if (int(lane) == i) mine = word;
  }
  if (int(lane) < n) planes[(uint64_t(lane) * rows + r) * wpr + w] = mine;
}

// Per-row granularity: one block per row (absmax reduce, then quantize+pack its words).
__global__ void __launch_bounds__(kThreads)
    quantize_rows_kernel(const double* __restrict__ x, uint64_t rows, uint64_t cols, int n,
                         uint32_t* __restrict__ planes, double* __restrict__ scales,
                         uint8_t* __restrict__ codes, int* __restrict__ flag) {
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
  if (threadIdx.x == 0) scales[r] = s;
  const uint64_t wpr = (cols + 31) / 32;
  for (uint64_t w = threadIdx.x >> 5; w < wpr; w += blockDim.x / 32) {
    quantize_pack_word(xrow, r, rows, cols, w, n, maxv, s, planes, codes);
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
                           const int* flag) {
  if (*flag) return;
  const int maxv = (1 << n) - 1;
  const double m = __longlong_as_double(static_cast<long long>(*amax_bits));
  const double s = m == 0.0 ? 1.0 : __ddiv_rn(m, double(maxv));
  if (blockIdx.x == 0 && threadIdx.x == 0) scales[0] = s;
  const uint64_t wpr = (cols + 31) / 32;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (gw >= rows * wpr) return;
  const uint64_t r = gw / wpr, w = gw % wpr;
  quantize_pack_word(x + r * cols, r, rows, cols, w, n, maxv, s, planes, codes);
}

unsigned blocks_for(uint64_t threads) {
  return static_cast<unsigned>((threads + kThreads - 1) / kThreads);
}

}  // namespace

cudaError_t launch_expand(const uint32_t* planes, uint64_t rows, uint64_t cols, int n,
                          uint8_t* codes, uint64_t kpad, int32_t* rowsum, cudaStream_t s) {
  const uint32_t wpr = static_cast<uint32_t>((cols + 31) / 32);
  const uint32_t tail = static_cast<uint32_t>(cols & 31);
  const uint32_t tail_mask = tail ? ((1u << tail) - 1u) : 0xffffffffu;
  const uint32_t kpad_words = static_cast<uint32_t>(kpad / 32);
  const int threads = kpad_words >= 256 ? 256 : (kpad_words >= 128 ? 128 : 64);
  expand_kernel<<<static_cast<unsigned>(rows), threads, 0, s>>>(
      planes, static_cast<uint32_t>(rows), wpr, n, tail_mask, codes, kpad_words, rowsum);
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
                                 cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  if (granularity == 1) {
    quantize_rows_kernel<<<static_cast<unsigned>(rows), kThreads, 0, s>>>(x, rows, cols, n,
                                                                          planes, scales, codes,
                                                                          flag);
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
                                                                     planes, scales, codes, flag);
  return cudaGetLastError();
}

// ---- tensor maps ------------------------------------------------------------------------------
CUresult encode_tmap_u8_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                           uint32_t box_inner, uint32_t box_outer) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr) {
      return CUDA_ERROR_NOT_FOUND;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {inner};  // bytes, for dim 1
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t elem_strides[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                elem_strides, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace apmm_b200
