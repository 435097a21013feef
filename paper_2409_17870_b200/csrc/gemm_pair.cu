// gemm_pair.cu -- K3 (large tiles): the WnAm bipolar-INT GEMM on a CTA PAIR
// (tcgen05 cta_group::2), 256 x 256 output tile per pair.
//
// Same arithmetic as gemm_tc.cu (one u8 x u8 kind::i8 MMA recovers every 2^(i+j)-weighted
// plane pair; rank-1 correction in the epilogue), but each MMA spans both SMs of a TPC:
// CTA r holds W rows [tm*256 + r*128, +128) (A) and X rows [tn*256 + r*128, +128) (B);
// the leader's tcgen05.mma.cta_group::2 (M=256, N=256, K=32) reads A and B from both
// CTAs' shared memory and writes a 128 x 256 s32 accumulator into each CTA's TMEM. Per
// SM this halves the operand bytes per MAC relative to the 1-SM 128x256 tile (32 KB per
// 128-K stage instead of 48 KB), which leaves room for 6 stages.
//
// Roles (both CTAs unless noted):
//   warp 0     TMA producer: own halves of A and B; completion bytes land on the LEADER's
//              full barrier (leader arms it with the pair's 64 KB)
//   warp 1     (leader) MMA issuer; tcgen05.commit multicast frees smem slots in both CTAs
//              and signals both CTAs' epilogues
//   warp 2     TMEM allocator (cta_group::2, 512 columns = 2 accumulator buffers)
//   warps 4-7  epilogue: tcgen05.ld -> rank-1 recovery (or fp64 dequant) -> 128B-swizzled
//              smem staging -> TMA bulk tensor store; arrive on the leader's tmem_empty
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace apmm_b200 {
namespace {

using namespace apmm_ptx;

constexpr int kHalf = 128;                   // rows of A and of B held per CTA
constexpr int kStages = 6;
constexpr int kAS = kHalf * kBK;             // 16 KB
constexpr int kStageBytes = 2 * kHalf * kBK; // A + B = 32 KB per CTA per stage
constexpr int kThreads = 256;
constexpr int kEpiBuf = 32 * 32 * 4;         // one 32x32 x 4B staging tile
constexpr uint32_t kTmemCols = 512;
constexpr int kSmemBytes = kStages * kStageBytes + 4 * 2 * kEpiBuf + 1024 + 256;
constexpr uint32_t kIdesc = idesc_i8_u8u8(2 * kHalf, kPairN);
constexpr uint32_t kIdescHalf = idesc_i8_u8u8(2 * kHalf, kPairN / 2);

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
  uint32_t coef_w, coef_x, c0;
  uint32_t tma_store;  // 1: epilogue stores through tmap_y
  uint32_t n_full;     // tiles [0, n_full) are 256 x 256; the remaining full tiles of the
                       // last partial wave run as two 256 x 128 halves each (CL == 2 only)
  unsigned long long* dbg;  // optional wait-cycle counters (APMM_DEBUG_WAITS), else null
  uint32_t peak_probe;      // APMM_PEAK_PROBE=1 (measurement only): no operand reloads
  // split-K (calls with too few tiles to fill the machine; CL == 2, int32 out): unit u =
  // (tile u / split of `ncols` feature rows, K blocks [ks*kb_per, +kb_per)); int32 partials
  // are TMA reduce-added into a Y zeroed by K1; the unit holding K block 0 adds the rank-1
  // recovery terms. 0 = off.
  uint32_t split, kb_per, ncols, tiles_n_split;
  unsigned long long* ts;   // APMM_PAIR_TS=1 (dev only): per-CTA phase timestamps, else null
  unsigned* colmax;         // dequant: per-column (or global) |v| max for the requantizer
  uint32_t colmax_global;
};

__device__ __forceinline__ unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct PUnit {
  uint32_t tm, col0, ncols, kb0, kb1;
  bool first;
};

// TMA reduce-add of a staged 32x32 int32 tile into Y (exact mod 2^32)
APMM_DEV void tma_reduce_add_2d(const void* tmap, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ uint32_t dequant_bits(uint32_t v, double sw, double sx) {
  return __float_as_uint(static_cast<float>(__dmul_rn(__dmul_rn(double(int(v)), sw), sx)));
}

// CL = 2: one CTA pair per cluster. CL = 4: two pairs per cluster computing vertically
// adjacent tiles (W rows tm and tm+1, same X rows): each X half is loaded once per cluster
// and multicast into both pairs (CTA q and q+2), cutting the L2 -> SMEM bytes per MAC by
// a quarter; a stage is released only when both pairs' MMAs have consumed it.
// Tile t of the persistent schedule: W row tile (256 rows), first X row, and X row count.
// Wave-quantization fix: with T full tiles on P pairs, the r = T mod P tiles of the last
// partial wave (r <= P/2) are split into 2r half-width tiles, so that wave costs half.
struct TileInfo {
  uint32_t tm, col0, ncols;
};
__device__ __forceinline__ TileInfo tile_info(uint32_t t, uint32_t tiles_m, uint32_t tiles_n,
                                             uint32_t n_full) {
  uint32_t tm, tn;
  if (t < n_full) {
    raster_tile(t, tiles_m, tiles_n, tm, tn);
    return {tm, tn * kPairN, kPairN};
  }
  const uint32_t h = t - n_full, f = n_full + (h >> 1);
  raster_tile(f, tiles_m, tiles_n, tm, tn);
  return {tm, tn * kPairN + (h & 1u) * (kPairN / 2), kPairN / 2};
}

__device__ __forceinline__ PUnit pair_unit(uint32_t t, const Params& p) {
  if (!p.split) {
    const TileInfo ti = tile_info(t, p.tiles_m, p.tiles_n, p.n_full);
    return {ti.tm, ti.col0, ti.ncols, 0u, p.kblocks, true};
  }
  const uint32_t tile = t / p.split, ks = t - tile * p.split;
  uint32_t tm, tn;
  raster_tile(tile, p.tiles_m, p.tiles_n_split, tm, tn);
  const uint32_t kb0 = ks * p.kb_per;
  const uint32_t kb1 = kb0 + p.kb_per < p.kblocks ? kb0 + p.kb_per : p.kblocks;
  return {tm, tn * p.ncols, p.ncols, kb0, kb1, ks == 0};
}

template <int CL>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_u8_pair_kernel(const __grid_constant__ CUtensorMap tmap_w,
                        const __grid_constant__ CUtensorMap tmap_x,
                        const __grid_constant__ CUtensorMap tmap_x64,
                        const __grid_constant__ CUtensorMap tmap_y, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  uint8_t* stages = smem;
  uint8_t* staging = smem + kStages * kStageBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + 4 * 2 * kEpiBuf);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tmem_full = empty_bar + kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  if (p.ts && threadIdx.x == 0) p.ts[blockIdx.x * 8 + 0] = gtime_ns();
  const uint32_t rank = cluster_ctarank();
  const uint32_t q = rank & 1u;              // role within the pair (0 = MMA leader)
  const uint32_t pr = rank >> 1;             // pair index within the cluster
  const uint32_t lead_rank = rank & ~1u;     // my pair's leader
  const bool leader = q == 0;
  const uint32_t cluster = blockIdx.x / CL;
  const uint32_t nclusters = gridDim.x / CL;
  constexpr uint32_t kPairs = CL / 2;
  const uint32_t tiles_mc = (p.tiles_m + kPairs - 1) / kPairs;  // cluster tiles along W rows
  const uint32_t num_tiles =
      CL == 2 ? (p.split ? p.tiles_m * p.tiles_n_split * p.split
                         : p.n_full + 2 * (p.tiles_m * p.tiles_n - p.n_full))
              : tiles_mc * p.tiles_n;
  constexpr uint16_t kAllMask = static_cast<uint16_t>((1u << CL) - 1u);
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2u * pr));

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_w);
    tma_prefetch_desc(&tmap_x);
    if (CL == 2) tma_prefetch_desc(&tmap_x64);
    if (p.tma_store) tma_prefetch_desc(&tmap_y);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kPairs);  // one MMA commit per pair
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: everything above overlapped the previous kernel; from here on we read the
  // operand workspace and write Y, so wait for the expand kernel (which itself completes
  // only after the previous GEMM). Then let the NEXT call's expand start on the spare
  // issue slots / registers of this SM while our tensor cores run.
  pdl_wait();
  if (threadIdx.x == 0) pdl_trigger();
  if (p.ts && threadIdx.x == 0) p.ts[blockIdx.x * 8 + 1] = gtime_ns();

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (elect_one()) {
      const uint64_t hint = policy_evict_last();
      uint32_t stage = 0, phase = 0, loaded = 0;
      for (uint32_t t = cluster; t < num_tiles; t += nclusters) {
        const PUnit un = CL == 2 ? pair_unit(t, p)
                                 : PUnit{(t % tiles_mc) * kPairs + pr, (t / tiles_mc) * kPairN,
                                         kPairN, 0u, p.kblocks, true};
        const TileInfo ti{un.tm, un.col0, un.ncols};
        const uint32_t tm = ti.tm;
        const bool half = ti.ncols != kPairN;
        for (uint32_t kb = un.kb0; kb < un.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (p.peak_probe && loaded >= kStages) {
            // measurement mode (APMM_PEAK_PROBE=1, results wrong): after one ring fill the
            // stages are re-used without loads -> the tcgen05 kind::i8 pipe's own ceiling
            // with this kernel's schedule, MMA issue and epilogue
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 0);
            if (++stage == kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          ++loaded;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], half ? 3 * kAS : 2 * kStageBytes);
          const uint32_t fb = mapa(smem_u32(&full_bar[stage]), lead_rank);
          uint8_t* st = stages + stage * kStageBytes;
          tma_load_2d_pair(st, &tmap_w, fb, int32_t(kb * kBK), int32_t(tm * 2 * kHalf + q * kHalf),
                           hint);
          if (CL == 2) {
            if (half) {
              tma_load_2d_pair(st + kAS, &tmap_x64, fb, int32_t(kb * kBK),
                               int32_t(ti.col0 + q * (kHalf / 2)), hint);
            } else {
              tma_load_2d_pair(st + kAS, &tmap_x, fb, int32_t(kb * kBK),
                               int32_t(ti.col0 + q * kHalf), hint);
            }
          } else if ((kb & 1u) == pr) {  // the pairs take turns loading the shared X half
            tma_load_2d_pair_mc(st + kAS, &tmap_x, fb, int32_t(kb * kBK),
                                int32_t(ti.col0 + q * kHalf),
                                static_cast<uint16_t>((1u << q) | (1u << (q + 2))), hint);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only) ----------------
    if (leader && elect_one()) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      unsigned long long w_full = 0, w_tmem = 0, t_begin = clock64();
      for (uint32_t t = cluster; t < num_tiles; t += nclusters) {
        unsigned long long c0 = p.dbg ? clock64() : 0;
        (void)c0;
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        if (p.dbg) w_tmem += clock64() - c0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kPairN;
        const PUnit un = CL == 2 ? pair_unit(t, p) : PUnit{0u, 0u, kPairN, 0u, p.kblocks, true};
        const uint32_t idesc = un.ncols != kPairN ? kIdescHalf : kIdesc;
        for (uint32_t kb = un.kb0; kb < un.kb1; ++kb) {
          c0 = p.dbg ? clock64() : 0;
          mbar_wait(&full_bar[stage], phase);
          if (p.dbg) w_full += clock64() - c0;
          if (p.ts && t == cluster && kb == un.kb0) p.ts[blockIdx.x * 8 + 2] = gtime_ns();
          tc_fence_after();
          const uint32_t st = smem_u32(stages + stage * kStageBytes);
          const uint64_t adesc = umma_desc_sw128(st);
          const uint64_t bdesc = umma_desc_sw128(st + kAS);
#pragma unroll
          for (uint32_t k = 0; k < kBK / 32; ++k) {
            mma_i8_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != un.kb0) || k != 0);
          }
          mma_commit_pair_mc(&empty_bar[stage], kAllMask);  // frees the slot in every CTA
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair_mc(&tmem_full[acc], pair_mask);
        if (p.ts) p.ts[blockIdx.x * 8 + 3] = gtime_ns();  // last write = last unit issued
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
      if (p.dbg) {
        atomicAdd(p.dbg + 0, w_full);
        atomicAdd(p.dbg + 1, w_tmem);
        atomicAdd(p.dbg + 2, clock64() - t_begin);
        atomicAdd(p.dbg + 3, 1ull);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs) ----------------
    const uint32_t wq = warp & 3;
    uint32_t acc = 0, acc_phase = 0, nbuf = 0;
    const uint64_t store_hint = policy_evict_first();  // Y streams out; keep operands in L2
    for (uint32_t t = cluster; t < num_tiles; t += nclusters) {
      const PUnit un = CL == 2 ? pair_unit(t, p)
                               : PUnit{(t % tiles_mc) * kPairs + pr, (t / tiles_mc) * kPairN,
                                       kPairN, 0u, p.kblocks, true};
      const TileInfo ti{un.tm, un.col0, un.ncols};
      const uint32_t tm = ti.tm;
      const uint32_t row0 = tm * 2 * kHalf + q * kHalf + wq * 32;
      const uint32_t row = row0 + lane;
      const bool row_ok = row < p.rows_w;
      const uint32_t rsw = row_ok ? static_cast<uint32_t>(__ldg(p.rowsum_w + row)) : 0u;
      // split-K: the unit holding K block 0 adds the whole rank-1 term (full-K rowsums)
      const uint32_t row_term = un.first ? p.c0 - p.coef_w * rsw : 0u;
      const uint32_t coef_x = un.first ? p.coef_x : 0u;
      double sw = 0.0;
      if (p.yf) sw = p.gran_w ? (row_ok ? p.s_w[row] : 0.0) : p.s_w[0];

      // this tile's rowsum(U_x) into registers BEFORE waiting for the accumulator (lane l
      // holds columns 8l..8l+7; chunk c's column j is a shuffle from lane 4c + j/8): the
      // per-chunk global loads were serialised L2 round trips (~0.8 us each) exposed on a
      // CTA's last tile (APMM_PAIR_TS timeline)
      int4 rsx_lo = make_int4(0, 0, 0, 0), rsx_hi = make_int4(0, 0, 0, 0);
      if (8u * lane < ti.ncols) {
        const int4* src = reinterpret_cast<const int4*>(p.rowsum_x + ti.col0 + 8u * lane);
        rsx_lo = __ldg(src);
        rsx_hi = __ldg(src + 1);
      }
      mbar_wait(&tmem_full[acc], acc_phase);
      tc_fence_after();
      const uint32_t t_addr = tmem_base + ((wq * 32u) << 16) + acc * kPairN;
#pragma unroll 1
      for (uint32_t c = 0; c < ti.ncols / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_addr + c * 32, r);
        tmem_ld_wait();
        const uint32_t col0 = ti.col0 + c * 32;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          // columns 4 j4 .. 4 j4 + 3 of the chunk: lane 4c + j4/2, half (j4 & 1)
          const uint32_t src_lane = 4u * c + (j4 >> 1);
          const int4 mine = (j4 & 1) ? rsx_hi : rsx_lo;
          int4 rs;
          rs.x = __shfl_sync(0xffffffffu, mine.x, src_lane);
          rs.y = __shfl_sync(0xffffffffu, mine.y, src_lane);
          rs.z = __shfl_sync(0xffffffffu, mine.z, src_lane);
          rs.w = __shfl_sync(0xffffffffu, mine.w, src_lane);
          r[4 * j4 + 0] = 4u * r[4 * j4 + 0] + row_term - coef_x * uint32_t(rs.x);
          r[4 * j4 + 1] = 4u * r[4 * j4 + 1] + row_term - coef_x * uint32_t(rs.y);
          r[4 * j4 + 2] = 4u * r[4 * j4 + 2] + row_term - coef_x * uint32_t(rs.z);
          r[4 * j4 + 3] = 4u * r[4 * j4 + 3] + row_term - coef_x * uint32_t(rs.w);
        }
        if (p.yf) {
          if (p.gran_x) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const uint32_t cj = col0 + j < p.rows_x ? col0 + j : 0;
              r[j] = dequant_bits(r[j], sw, __ldg(p.s_x + cj));
            }
          } else {
            const double sx = p.s_x[0];
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = dequant_bits(r[j], sw, sx);
          }
          if (p.colmax) {
            uint32_t f[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) f[j] = row_ok && col0 + j < p.rows_x ? r[j] : 0u;
            colmax_warp(f, lane, col0, p.rows_x, p.colmax, p.colmax_global != 0);
          }
        }
        if (p.tma_store) {
          uint8_t* buf = staging + (wq * 2 + nbuf) * kEpiBuf;
          nbuf ^= 1;
          if (lane == 0) bulk_wait_read<1>();  // the store that last read `buf` is done
          __syncwarp();
          const uint32_t base = smem_u32(buf) + lane * 128u;
#pragma unroll
          for (uint32_t ch = 0; ch < 8; ++ch) {  // SWIZZLE_128B: 16B chunk ch -> ch ^ (row & 7)
            st_shared_v4(base + ((ch ^ (lane & 7u)) << 4), r[4 * ch], r[4 * ch + 1],
                         r[4 * ch + 2], r[4 * ch + 3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (p.split) {
              tma_reduce_add_2d(&tmap_y, buf, int32_t(col0), int32_t(row0));
            } else {
              tma_store_2d(&tmap_y, buf, int32_t(col0), int32_t(row0), store_hint);
            }
            bulk_commit();
          }
        } else if (row_ok && col0 < p.rows_x) {
          uint32_t* dst = (p.y ? reinterpret_cast<uint32_t*>(p.y) : reinterpret_cast<uint32_t*>(p.yf)) +
                          uint64_t(row) * p.rows_x + col0;
#pragma unroll
          for (uint32_t j = 0; j < 32; ++j) {
            if (col0 + j < p.rows_x) dst[j] = r[j];
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa(smem_u32(&tmem_empty[acc]), lead_rank));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    // the staging buffers must have been read before the CTA exits; the stores themselves
    // complete with the grid (as CUTLASS's tma_store_wait), so no write round trip here
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
    if (p.ts && lane == 0 && warp == 4) p.ts[blockIdx.x * 8 + 4] = gtime_ns();
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
}

}  // namespace

cudaError_t launch_gemm_pair(const GemmArgs& a, cudaStream_t s, int* launches, bool split_k) {
  CUtensorMap tw, tx, tx64, ty;
  if (encode_tmap_2d(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.codes_w, a.kpad, a.rows_w, a.kpad,
                     kBK, kHalf) != CUDA_SUCCESS ||
      encode_tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.codes_x, a.kpad, a.rows_x, a.kpad,
                     kBK, kHalf) != CUDA_SUCCESS ||
      encode_tmap_2d(&tx64, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.codes_x, a.kpad, a.rows_x, a.kpad,
                     kBK, kHalf / 2) != CUDA_SUCCESS) {
    return cudaErrorInvalidValue;
  }
  void* out = a.y ? static_cast<void*>(a.y) : static_cast<void*>(a.yf);
  const bool tma_store = (a.rows_x % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  if (tma_store) {
    if (encode_tmap_2d(&ty, a.y ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                       4, out, a.rows_x, a.rows_w, a.rows_x * 4, 32, 32) != CUDA_SUCCESS) {
      return cudaErrorInvalidValue;
    }
  } else {
    ty = tw;  // unused
  }
  static DeviceBits attr_set;
  const int dev = current_device();
  if (!attr_set.test(dev)) {
    cudaError_t e = cudaFuncSetAttribute(gemm_u8_pair_kernel<2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (e == cudaSuccess) {
      e = cudaFuncSetAttribute(gemm_u8_pair_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               kSmemBytes);
    }
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
  p.tiles_m = static_cast<uint32_t>((a.rows_w + 2 * kHalf - 1) / (2 * kHalf));
  p.tiles_n = static_cast<uint32_t>((a.rows_x + kPairN - 1) / kPairN);
  const uint32_t A = (1u << a.n_w) - 1u, B = (1u << a.n_x) - 1u;
  p.coef_w = 2u * B;
  p.coef_x = 2u * A;
  p.c0 = static_cast<uint32_t>(a.k_logical) * A * B;
  p.tma_store = tma_store ? 1u : 0u;
  p.dbg = a.dbg;
  p.colmax = a.colmax;
  p.colmax_global = a.colmax_global ? 1u : 0u;
  static const uint32_t peak_probe = APMM_DEV_ENV("APMM_PEAK_PROBE") ? 1u : 0u;
  p.peak_probe = peak_probe;
  static const bool want_ts = APMM_DEV_ENV("APMM_PAIR_TS") != nullptr;
  static unsigned long long* ts_buf = nullptr;
  if (want_ts) {
    if (!ts_buf) cudaMalloc(&ts_buf, 512 * 8 * sizeof(unsigned long long));
    cudaMemsetAsync(ts_buf, 0, 512 * 8 * sizeof(unsigned long long), s);
    p.ts = ts_buf;
  }
  if (a.trace) p.ts = a.trace;  // dev launch trace (APMM_TRACE)
  // clusters of 4 (X multicast across two pairs) when there are enough cluster tiles to
  // fill the machine, else plain pairs. APMM_PAIR_CLUSTER=2|4 forces one (testing).
  static const int forced = [] {
    const char* f = APMM_DEV_ENV("APMM_PAIR_CLUSTER");
    return f ? std::atoi(f) : 0;
  }();
  const uint32_t quad_tiles = ((p.tiles_m + 1) / 2) * p.tiles_n;
  const uint32_t max_quads = static_cast<uint32_t>(a.num_sms / 4);
  // Default: pairs. Clusters of 4 cut L2 bytes by a quarter but only 33 fit (GPC
  // boundaries -> 132 SMs) and measured no faster (profiles/r01_notes.md).
  const int cl = forced == 2 || forced == 4 ? forced : 2;
  (void)max_quads;
  const uint32_t full_tiles = p.tiles_m * p.tiles_n;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = static_cast<unsigned>(cl);
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  // persistent grid = the clusters that can be co-resident (clusters cannot straddle GPCs,
  // so for 4-CTA clusters this can be fewer than num_sms / 4)
  static int max_active_dev[kMaxDevices][5] = {};
  int* max_active = max_active_dev[dev];
  if (!max_active[cl]) {
    cfg.gridDim = dim3(static_cast<unsigned>(a.num_sms / cl * cl));
    int n = 0;
    cudaError_t oe = cl == 4 ? cudaOccupancyMaxActiveClusters(&n, gemm_u8_pair_kernel<4>, &cfg)
                             : cudaOccupancyMaxActiveClusters(&n, gemm_u8_pair_kernel<2>, &cfg);
    max_active[cl] = (oe == cudaSuccess && n > 0) ? n : a.num_sms / cl;
    if (APMM_DEV_ENV("APMM_DEBUG_PLAN")) {
      std::fprintf(stderr, "[apmm pair] cluster %d: %d co-resident clusters\n", cl, max_active[cl]);
    }
  }
  const uint32_t max_clusters = static_cast<uint32_t>(max_active[cl]);
  // last-wave split (pairs only): r = T mod P tiles become 2r half-width tiles if r <= P/2
  p.n_full = full_tiles;
  if (cl == 2 && APMM_DEV_ENV("APMM_NO_TAIL_SPLIT") == nullptr) {
    const uint32_t r = full_tiles % max_clusters;
    if (r != 0 && 2 * r <= max_clusters) p.n_full = full_tiles - r;
  }
  uint32_t tiles = cl == 4 ? quad_tiles : p.n_full + 2 * (full_tiles - p.n_full);
  if (split_k && cl == 2) {
    // too few tiles for the machine: tiles of 128 (M_tok <= 128) or 256 feature rows, K split
    // so that the units fill the co-resident pairs; Y was zeroed by K1
    p.ncols = a.rows_x <= 128 ? 128u : 256u;
    p.tiles_n_split = static_cast<uint32_t>((a.rows_x + p.ncols - 1) / p.ncols);
    const uint32_t t2 = p.tiles_m * p.tiles_n_split;
    uint32_t sk = max_clusters / (t2 ? t2 : 1);
    const uint32_t max_s = p.kblocks / 4 > 0 ? p.kblocks / 4 : 1;  // >= 4 K blocks per unit
    sk = sk < 1 ? 1 : (sk > max_s ? max_s : sk);
    p.kb_per = (p.kblocks + sk - 1) / sk;
    p.split = (p.kblocks + p.kb_per - 1) / p.kb_per;
    tiles = t2 * p.split;
    if (APMM_DEV_ENV("APMM_DEBUG_PLAN")) {
      std::fprintf(stderr, "[apmm pair] split-K: %u tiles of %u cols x %u K splits of %u blocks\n",
                   t2, p.ncols, p.split, p.kb_per);
    }
  }
  const uint32_t clusters = tiles < max_clusters ? tiles : max_clusters;
  cfg.gridDim = dim3(cl * clusters);
  cudaError_t e = cl == 4 ? cudaLaunchKernelEx(&cfg, gemm_u8_pair_kernel<4>, tw, tx, tx64, ty, p)
                          : cudaLaunchKernelEx(&cfg, gemm_u8_pair_kernel<2>, tw, tx, tx64, ty, p);
  *launches += 1;
  if (want_ts && e == cudaSuccess) {  // dev only: per-phase CTA timeline (us from first start)
    unsigned long long h[512 * 8];
    const unsigned g = cfg.gridDim.x;
    cudaStreamSynchronize(s);
    cudaMemcpy(h, ts_buf, g * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull;
    for (unsigned b = 0; b < g; ++b) t0 = h[b * 8] && h[b * 8] < t0 ? h[b * 8] : t0;
    const char* names[5] = {"start", "pdl_wait", "first_full", "last_issue", "epi_done"};
    for (int k = 0; k < 5; ++k) {
      double mn = 1e30, mx = 0, sum = 0;
      unsigned cnt = 0;
      for (unsigned b = 0; b < g; ++b) {
        if (!h[b * 8 + k]) continue;
        const double v = (h[b * 8 + k] - t0) * 1e-3;
        mn = v < mn ? v : mn;
        mx = v > mx ? v : mx;
        sum += v;
        ++cnt;
      }
      std::fprintf(stderr, "[apmm pair ts] %-10s min %7.2f avg %7.2f max %7.2f us (%u CTAs)\n",
                   names[k], cnt ? mn : 0.0, cnt ? sum / cnt : 0.0, mx, cnt);
    }
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace apmm_b200
