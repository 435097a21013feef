// expand.cuh -- the planes -> u8-code expansion of one operand row (K1's per-warp work),
// shared by the expand kernel (prep.cu) and the in-kernel feature prep of the split-K
// weight-plane GEMM (gemm_fused.cu).
//
// One warp per row, lanes striding over the 32-column words. A lane turns the n plane words
// of a 32-column group into 32 code bytes with an 8x8 bit transpose done SIMD across the 4
// byte lanes of a 32-bit register (3 delta-swap stages, ~60 ALU ops for any n <= 8; rows
// i >= n are compile-time zero and fold away). The transpose leaves code(k = 8b + c) in byte
// b of output word c, i.e. the 32 codes of a group are stored in the K order (c, b) -> 4c + b
// instead of 8b + c. Both operands use the same order, and sum_k u_w(k) u_x(k) is invariant
// under a common permutation of k, so the GEMM result is unchanged; the zero padding lanes
// stay zero. rowsum(U) = sum_k u_k = sum_i 2^i popc(plane_i) comes straight from the planes.
#pragma once
#include <cstdint>

namespace apmm_b200 {
namespace xpd {

struct ExpandOperand {
  const uint32_t* planes;
  uint8_t* codes;
  int32_t* rowsum;
  uint32_t rows;
  uint32_t rows_pad;  // rowsum[rows, rows_pad) is zeroed (GEMM epilogue reads whole tiles)
  int n;
  int stream_store;   // 1: codes stored evict-first (st.global.cs), see launch_expand
};

constexpr int kExpandUnroll = 4;     // words per lane with loads in flight together

// 8x8 bit transpose inside every byte lane of x[0..7] (row i = plane i). Each swap is the
// select form  b' = (b & ~m) | ((a >> s) & m),  a' = (a & ~(m << s)) | ((b << s) & (m << s)):
// 4 ops per pair (SHF + LOP3 each), 12 pairs.
__device__ __forceinline__ void swap_sel(uint32_t& a, uint32_t& b, int s, uint32_t m) {
  const uint32_t na = (a & ~(m << s)) | ((b << s) & (m << s));
  b = (b & ~m) | ((a >> s) & m);
  a = na;
}

__device__ __forceinline__ void transpose8(uint32_t (&x)[8]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) swap_sel(x[i], x[i + 4], 4, 0x0F0F0F0Fu);
#pragma unroll
  for (int i = 0; i < 8; i += 4) {
    swap_sel(x[i], x[i + 2], 2, 0x33333333u);
    swap_sel(x[i + 1], x[i + 3], 2, 0x33333333u);
  }
#pragma unroll
  for (int i = 0; i < 8; i += 2) swap_sel(x[i], x[i + 1], 1, 0x55555555u);
}

// rowsum only (operand expanded elsewhere): sum_i 2^i popc(plane_i), lanes over words.
template <int N>
__device__ __forceinline__ int32_t rowsum_row(const ExpandOperand& op, uint32_t r, uint32_t wpr,
                                              uint32_t tail_mask, uint32_t lane) {
  int32_t sum = 0;
  const uint32_t* src = op.planes + uint64_t(r) * wpr;
  const uint64_t pstride = uint64_t(op.rows) * wpr;
  for (uint32_t w = lane; w < wpr; w += 32) {
    const uint32_t mask = w == wpr - 1 ? tail_mask : 0xffffffffu;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i < op.n) sum += __popc(__ldg(src + i * pstride + w) & mask) << i;
    }
  }
  return sum;
}

template <int N>
__device__ __forceinline__ int32_t expand_row(const ExpandOperand& op, uint32_t r, uint32_t wpr,
                                              uint32_t tail_mask, uint32_t kpad_words,
                                              uint32_t lane) {
  int32_t sum = 0;
  uint8_t* dst_row = op.codes + uint64_t(r) * kpad_words * 32u;
  const uint32_t* src = op.planes + uint64_t(r) * wpr;
  const uint64_t pstride = uint64_t(op.rows) * wpr;
  for (uint32_t w0 = 0; w0 < kpad_words; w0 += 32 * kExpandUnroll) {
    uint32_t x[kExpandUnroll][8];
#pragma unroll
    for (int u = 0; u < kExpandUnroll; ++u) {  // all loads first (memory-level parallelism)
      const uint32_t w = w0 + lane + 32 * u;
      const uint32_t mask = w < wpr ? (w == wpr - 1 ? tail_mask : 0xffffffffu) : 0u;
      const uint32_t wc = w < wpr ? w : 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) x[u][i] = i < N ? (__ldg(src + i * pstride + wc) & mask) : 0u;
    }
#pragma unroll
    for (int u = 0; u < kExpandUnroll; ++u) {
      const uint32_t w = w0 + lane + 32 * u;
#pragma unroll
      for (int i = 0; i < N; ++i) sum += __popc(x[u][i]) << i;
      transpose8(x[u]);
      if (w < kpad_words) {
        uint4* d = reinterpret_cast<uint4*>(dst_row + uint64_t(w) * 32u);
        if (op.stream_store) {
          __stcs(d, make_uint4(x[u][0], x[u][1], x[u][2], x[u][3]));
          __stcs(d + 1, make_uint4(x[u][4], x[u][5], x[u][6], x[u][7]));
        } else {
          d[0] = make_uint4(x[u][0], x[u][1], x[u][2], x[u][3]);
          d[1] = make_uint4(x[u][4], x[u][5], x[u][6], x[u][7]);
        }
      }
    }
  }
  return sum;
}

__device__ __forceinline__ void expand_one(const ExpandOperand& op, uint32_t r, uint32_t wpr,
                                           uint32_t tail_mask, uint32_t kpad_words,
                                           uint32_t lane) {
  int32_t sum = 0;
  if (op.codes == nullptr) {
    switch (op.n) {
      case 1: sum = rowsum_row<1>(op, r, wpr, tail_mask, lane); break;
      case 2: sum = rowsum_row<2>(op, r, wpr, tail_mask, lane); break;
      case 3: sum = rowsum_row<3>(op, r, wpr, tail_mask, lane); break;
      case 4: sum = rowsum_row<4>(op, r, wpr, tail_mask, lane); break;
      default: sum = rowsum_row<8>(op, r, wpr, tail_mask, lane); break;
    }
  } else switch (op.n) {
    case 1: sum = expand_row<1>(op, r, wpr, tail_mask, kpad_words, lane); break;
    case 2: sum = expand_row<2>(op, r, wpr, tail_mask, kpad_words, lane); break;
    case 3: sum = expand_row<3>(op, r, wpr, tail_mask, kpad_words, lane); break;
    case 4: sum = expand_row<4>(op, r, wpr, tail_mask, kpad_words, lane); break;
    case 5: sum = expand_row<5>(op, r, wpr, tail_mask, kpad_words, lane); break;
    case 6: sum = expand_row<6>(op, r, wpr, tail_mask, kpad_words, lane); break;
    case 7: sum = expand_row<7>(op, r, wpr, tail_mask, kpad_words, lane); break;
    default: sum = expand_row<8>(op, r, wpr, tail_mask, kpad_words, lane); break;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) op.rowsum[r] = sum;
}

// The same with the plane count fixed at compile time (single-operand expansion launches:
// a fraction of expand_one's code, which matters for short launches -- instruction-cache
// misses were their top stall, profiles/r02_notes.md).
template <int N>
__device__ __forceinline__ void expand_one_n(const ExpandOperand& op, uint32_t r, uint32_t wpr,
                                             uint32_t tail_mask, uint32_t kpad_words,
                                             uint32_t lane) {
  int32_t sum = op.codes == nullptr ? rowsum_row<N>(op, r, wpr, tail_mask, lane)
                                    : expand_row<N>(op, r, wpr, tail_mask, kpad_words, lane);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) op.rowsum[r] = sum;
}

}  // namespace xpd
}  // namespace apmm_b200
