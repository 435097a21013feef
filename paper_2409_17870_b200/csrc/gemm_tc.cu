// gemm_tc.cu -- K3: the WnAm bipolar-INT GEMM on sm_100a 5th-gen tensor cores.
//
// Replaces the CPU plane-pair loop of matmul_ap (reference kernel.cpp:187-254). Instead of
// n_w*n_x binary plane products (the paper's BMMA formulation -- sm_100a has no b1 tensor
// pipe), all plane pairs are recovered INSIDE one u8 x u8 tcgen05 MMA:
// with unsigned codes u = sum_i 2^i b_i and bipolar value v = 2u - (2^n - 1),
//
//   Y = sum_ij 2^(i+j) Y^(ij) = 4 U_w U_x^T - 2B rowsum(U_w) 1^T - 2A 1 rowsum(U_x)^T + K A B
//
// (A = 2^n_w - 1, B = 2^n_x - 1, K the logical depth; zero K padding has u = 0 and drops
// out). The MMA accumulates U_w U_x^T exactly in s32 TMEM (max K*255^2 < 2^31 whenever the
// reference's overflow_bound admits the shape), and the epilogue applies the rank-1
// correction in wrapping u32 arithmetic -- exact because the true Y fits in int32. So no
// plane-pair intermediate ever exists, in HBM or on chip.
//
// Structure (one CTA per SM, persistent, warp-specialised):
//   warp 0      TMA producer: 128x128 B (W codes) + 256x128 B (X codes) per stage,
//               SWIZZLE_128B, 4-stage mbarrier ring
//   warp 1      MMA issuer: 4 x tcgen05.mma.kind::i8 (M=128, N=256, K=32) per stage,
//               accumulator double-buffered in TMEM (2 x 256 columns)
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld -> rank-1 correction (or fp64 dequant) -> st.global
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace apmm_b200 {
namespace {

using namespace apmm_ptx;

constexpr int kStages = 4;
constexpr int kAStage = kBM * kBK;  // 16 KB
constexpr int kBStage = kBN * kBK;  // 32 KB
constexpr int kThreads = 256;
constexpr uint32_t kTmemCols = 2 * kBN;  // two accumulator buffers
constexpr int kSmemBytes = kStages * (kAStage + kBStage) + 1024 /*align*/ + 256 /*bars*/;
constexpr uint32_t kIdesc = idesc_i8_u8u8(kBM, kBN);

struct Params {
  const int32_t* rowsum_w;
  const int32_t* rowsum_x;
  int32_t* y;
  float* yf;
  const double* s_w;
  const double* s_x;
  int gran_w, gran_x;
  uint32_t rows_w, rows_x;
  uint32_t kblocks;
  uint32_t tiles_m, tiles_n;
  uint32_t coef_w;  // 2*(2^n_x - 1): multiplies rowsum_w
  uint32_t coef_x;  // 2*(2^n_w - 1): multiplies rowsum_x
  uint32_t c0;      // K*(2^n_w-1)*(2^n_x-1) mod 2^32
  unsigned* colmax;         // dequant: per-column (or global) |v| max for the requantizer
  uint32_t colmax_global;
};

__global__ void __launch_bounds__(kThreads, 1)
    gemm_u8_tc_kernel(const __grid_constant__ CUtensorMap tmap_w,
                      const __grid_constant__ CUtensorMap tmap_x, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for the SWIZZLE_128B atoms.
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  uint8_t* sm_a = smem;
  uint8_t* sm_b = smem + kStages * kAStage;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm_b + kStages * kBStage);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tmem_full = empty_bar + kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t num_tiles = p.tiles_m * p.tiles_n;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], 4);  // one arrival per epilogue warp
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // see gemm_pair.cu: expand done (and, through it, the previous GEMM)
  if (threadIdx.x == 0) pdl_trigger();

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      const uint64_t hint = policy_evict_last();  // operands are re-read by many tiles
      uint32_t stage = 0, phase = 0;
      for (uint32_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        uint32_t tm, tn;
        raster_tile(t, p.tiles_m, p.tiles_n, tm, tn);
        for (uint32_t kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], kAStage + kBStage);
          tma_load_2d(sm_a + stage * kAStage, &tmap_w, &full_bar[stage], int32_t(kb * kBK),
                      int32_t(tm * kBM), hint);
          tma_load_2d(sm_b + stage * kBStage, &tmap_x, &full_bar[stage], int32_t(kb * kBK),
                      int32_t(tn * kBN), hint);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (elect_one()) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      for (uint32_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        for (uint32_t kb = 0; kb < p.kblocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint64_t adesc = umma_desc_sw128(smem_u32(sm_a + stage * kAStage));
          const uint64_t bdesc = umma_desc_sw128(smem_u32(sm_b + stage * kBStage));
#pragma unroll
          for (uint32_t k = 0; k < kBK / 32; ++k) {
            // +32 bytes of K inside the swizzle row == +2 in the (addr>>4) field
            mma_i8(d_tmem, adesc + 2 * k, bdesc + 2 * k, kIdesc, (kb | k) != 0);
          }
          mma_commit(&empty_bar[stage]);  // frees the smem slot when these MMAs finish
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        mma_commit(&tmem_full[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const uint32_t q = warp & 3;  // TMEM lane quadrant this warp may access
    uint32_t acc = 0, acc_phase = 0;
    for (uint32_t t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      uint32_t tm, tn;
        raster_tile(t, p.tiles_m, p.tiles_n, tm, tn);
      const uint32_t row = tm * kBM + q * 32 + lane;
      const bool row_ok = row < p.rows_w;
      const uint32_t rsw = row_ok ? static_cast<uint32_t>(__ldg(p.rowsum_w + row)) : 0u;
      const uint32_t row_term = p.c0 - p.coef_w * rsw;  // wrapping u32
      double sw = 0.0;
      if (p.yf) sw = p.gran_w ? p.s_w[row_ok ? row : 0] : p.s_w[0];

      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_addr = tmem_base + ((q * 32u) << 16) + acc * kBN;
#pragma unroll 1
      for (uint32_t c = 0; c < kBN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_addr + c * 32, r);
        tmem_ld_wait();
        const uint32_t col0 = tn * kBN + c * 32;
        const int4* rsx4 = reinterpret_cast<const int4*>(p.rowsum_x + col0);
        uint32_t v[32];
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const int4 rs = __ldg(rsx4 + j4);
          v[4 * j4 + 0] = 4u * r[4 * j4 + 0] + row_term - p.coef_x * uint32_t(rs.x);
          v[4 * j4 + 1] = 4u * r[4 * j4 + 1] + row_term - p.coef_x * uint32_t(rs.y);
          v[4 * j4 + 2] = 4u * r[4 * j4 + 2] + row_term - p.coef_x * uint32_t(rs.z);
          v[4 * j4 + 3] = 4u * r[4 * j4 + 3] + row_term - p.coef_x * uint32_t(rs.w);
        }
        if (row_ok && col0 < p.rows_x) {
          const uint64_t off = uint64_t(row) * p.rows_x + col0;
          if (p.y) {
            int32_t* dst = p.y + off;
            if (col0 + 32 <= p.rows_x && (p.rows_x % 4 == 0)) {
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                reinterpret_cast<int4*>(dst)[j4] =
                    make_int4(int(v[4 * j4]), int(v[4 * j4 + 1]), int(v[4 * j4 + 2]),
                              int(v[4 * j4 + 3]));
              }
            } else {
#pragma unroll
              for (uint32_t j = 0; j < 32; ++j) {
                if (col0 + j < p.rows_x) dst[j] = int(v[j]);
              }
            }
          } else {
            float* dst = p.yf + off;
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) {
              const double sx = p.gran_x ? p.s_x[col0 + j < p.rows_x ? col0 + j : 0] : p.s_x[0];
              const float fv = static_cast<float>(__dmul_rn(__dmul_rn(double(int(v[j])), sw), sx));
              v[j] = col0 + j < p.rows_x ? __float_as_uint(fv) : 0u;
              if (col0 + j < p.rows_x) dst[j] = fv;
            }
          }
        }
        __syncwarp();
        if (p.colmax) {
          if (!(row_ok && col0 < p.rows_x)) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0u;
          }
          colmax_warp(v, lane, col0, p.rows_x, p.colmax, p.colmax_global != 0);
        }
        __syncwarp();  // reconverge before the next .sync.aligned tcgen05.ld
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<kTmemCols>(tmem_base);
}

}  // namespace

cudaError_t launch_gemm_tc(const GemmArgs& a, cudaStream_t s, int* launches) {
  CUtensorMap tw, tx;
  if (encode_tmap_2d(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.codes_w, a.kpad, a.rows_w, a.kpad,
                     kBK, kBM) != CUDA_SUCCESS ||
      encode_tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.codes_x, a.kpad, a.rows_x, a.kpad,
                     kBK, kBN) != CUDA_SUCCESS) {
    return cudaErrorInvalidValue;
  }
  static DeviceBits attr_set;
  const int dev = current_device();
  if (!attr_set.test(dev)) {
    cudaError_t e = cudaFuncSetAttribute(gemm_u8_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set.set(dev);
  }
  Params p{};
  p.rowsum_w = a.rowsum_w;
  p.rowsum_x = a.rowsum_x;
  p.y = a.y;
  p.yf = a.yf;
  p.s_w = a.s_w;
  p.s_x = a.s_x;
  p.gran_w = a.gran_w;
  p.gran_x = a.gran_x;
  p.rows_w = static_cast<uint32_t>(a.rows_w);
  p.rows_x = static_cast<uint32_t>(a.rows_x);
  p.kblocks = static_cast<uint32_t>(a.kpad / kBK);
  p.tiles_m = static_cast<uint32_t>((a.rows_w + kBM - 1) / kBM);
  p.tiles_n = static_cast<uint32_t>((a.rows_x + kBN - 1) / kBN);
  const uint32_t A = (1u << a.n_w) - 1u, B = (1u << a.n_x) - 1u;
  p.coef_w = 2u * B;
  p.coef_x = 2u * A;
  p.c0 = static_cast<uint32_t>(a.k_logical) * A * B;  // wraps mod 2^32 by design
  p.colmax = a.colmax;
  p.colmax_global = a.colmax_global ? 1u : 0u;
  const uint32_t tiles = p.tiles_m * p.tiles_n;
  const uint32_t grid = tiles < uint32_t(a.num_sms) ? tiles : uint32_t(a.num_sms);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_u8_tc_kernel, tw, tx, p);
  *launches += 1;
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace apmm_b200
