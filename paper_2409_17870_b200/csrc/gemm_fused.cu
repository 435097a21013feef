// gemm_fused.cu -- K3f: the WnAm bipolar-INT GEMM on a CTA pair with the WEIGHT bit planes
// expanded on chip (the paper's "bit-plane preprocessing in the tile").
//
// Same pair schedule, TMEM double buffer and epilogue as gemm_pair.cu, but operand A (the
// weight rows) is never materialised as u8 codes in HBM/L2. Per 128-column K block:
//   * the TMA producer loads the raw reference-layout planes of this CTA's 128 weight rows,
//     box {4 words, 128 rows, n_w planes} = 2 KB per plane, into a raw ring slot;
//   * 4 transform warps (one thread per weight row) turn them into u8 codes with an 8x8 bit transpose inside every
//     byte lane (compile-time-zero planes fold away, so W1/W2 cost a fraction of W8), and
//     store them straight into the 128B-swizzled K-major layout UMMA reads -- the layout
//     TMA would have produced from the expanded codes;
//   * they fence the generic-proxy writes to the async proxy and arrive (cluster scope) on
//     the pair leader's full barrier, which also counts the TMA bytes of operand B (the
//     feature codes, expanded once per call by K1).
// L2 -> SMEM bytes per MAC for A drop from 8 to n_w bits per code: the large-tile kernel
// is L2-bandwidth bound (profiles/r01_notes.md), so this is what moves it toward the
// tensor-pipe roofline. The K order inside each 32-column group is the one K1 uses for X
// (byte 4c + b <- column 8b + c), so sum_k u_w(k) u_x(k) is unchanged.
//
// Roles (both CTAs unless noted): warp 0 TMA producer (B codes), warp 1 MMA issuer (leader),
// warp 2 TMEM allocator, warp 3 TMA producer (raw weight planes), warps 4-7 epilogue,
// warps 8-11 transform.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "expand.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace apmm_b200 {
namespace {

using namespace apmm_ptx;

constexpr int kHalf = 128;                    // rows of A and of B held per CTA
constexpr int kAS = kHalf * kBK;              // 16 KB of u8 codes per operand per stage
constexpr int kXformWarpsCfg = 8;  // transform warps (4: one thread per row; 8: two)
constexpr int kThreads = (8 + kXformWarpsCfg) * 32;
constexpr int kXformWarp0 = 8;                // first transform warp
constexpr int kXformWarps = kXformWarpsCfg;
constexpr int kWPT = 16 / kXformWarps;       // plane words (K/32 groups) per transform thread per block
constexpr int kEpiBuf = 32 * 32 * 4;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kIdesc = idesc_i8_u8u8(2 * kHalf, kPairN);
constexpr uint32_t kIdescHalf = idesc_i8_u8u8(2 * kHalf, kPairN / 2);
// A raw stage holds RB consecutive K blocks of the tile's 128 rows: TMA box
// {4*RB words, 128 rows, n_w planes}. RB > 1 makes each row segment of the box 16*RB bytes;
// with 16-byte segments (RB = 1) the TMA request count per K block doubled and the raw
// ring alone bounded the kernel at ~0.55 us per K block (ablation, 4096^3 W2A4).
__host__ __device__ constexpr int raw_rb(int nw) { return nw <= 4 ? 4 : 2; }
__host__ __device__ constexpr int raw_plane(int nw) { return kHalf * 16 * raw_rb(nw); }

// Two rings. The operand ring (A codes written by the transform warps + B codes by TMA,
// 32 KB a stage) feeds the MMA; the raw ring (the weight planes of one K block, n_w x 2 KB
// a stage) is filled by its own producer warp far ahead, so the plane loads' latency is
// off the operand ring's round trip (with a shared ring the kernel was latency bound:
// 0.56 us per stage at 4096^3 W2A4). Shared memory: rings + 32 KB epilogue staging +
// barriers, within the 227 KB opt-in.
__host__ __device__ constexpr int raw_bytes(int nw) { return nw * raw_plane(nw); }
constexpr int kOpStageBytes = 2 * kAS;
__host__ __device__ constexpr int op_stages(int nw) { return nw <= 2 ? 5 : 4; }
constexpr int kSmemCap = 232448 - 1024 - 1024 - 2048 - 4096;  // + 4 KB epilogue column terms  // 227 KB minus alignment slack, barriers and the static rowsum buffers
__host__ __device__ constexpr int raw_stages(int nw) {
  return (kSmemCap - op_stages(nw) * kOpStageBytes - 4 * 2 * kEpiBuf) / raw_bytes(nw) > 16
             ? 16
             : (kSmemCap - op_stages(nw) * kOpStageBytes - 4 * 2 * kEpiBuf) / raw_bytes(nw);
}
__host__ __device__ constexpr int smem_bytes(int nw) {
  return op_stages(nw) * kOpStageBytes + raw_stages(nw) * raw_bytes(nw) + 4 * 2 * kEpiBuf +
         1024 + 1024;
}

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
  uint32_t tma_store;
  uint32_t n_full;
  uint32_t n_w;        // runtime plane count (<= NW)
  uint32_t last_word;  // index of the last plane word of a row (wpr - 1)
  uint32_t tail_mask;  // valid bits of that word (reference padding is zero; masked anyway)
  // split-K mode (mid-size calls that cannot fill the machine with tiles): work unit u =
  // (tile u / split, K blocks [ks*kb_per, +kb_per) with ks = u % split); tiles are `ncols`
  // wide; partial sums are TMA reduce-added into a pre-zeroed Y, the rank-1 term by ks == 0.
  uint32_t split;   // 0: off (plain tiles, store epilogue)
  uint32_t kb_per, ncols, tiles_n_split;
  uint32_t ablate;  // dev only (APMM_FUSED_ABLATE, results wrong): 1 skip A stores, 2 skip B loads
  unsigned long long* dbg;  // APMM_DEBUG_WAITS=1: wait-cycle counters per role, else null
  unsigned long long* ts;   // dev launch trace (APMM_TRACE): [0] start [1] pdl_wait [4] end
  uint32_t early_w;         // PDL: weight-plane loads + transforms before the previous kernel ends
  uint32_t ts_clock;        // dev (APMM_TRACE_CLOCK): clock64 stamps inside the epilogue chunk loop
  // In-kernel feature prep (split mode; replaces the K1x launch): after griddepcontrol.wait
  // the epilogue warps of all CTAs expand X planes -> u8 codes + rowsum(U_x) (the layout K1
  // writes, read back by the B operand's TMA) and zero Y, then meet at a grid-wide barrier
  // (sense-reversing: count + generation) before B loads and reduce-adds.
  uint32_t xprep;
  const uint32_t* x_planes;
  uint8_t* x_codes;
  int32_t* x_rowsum;
  uint32_t rows_x_pad, n_x, wpr, kpad_words;
  uint4* y_zero;
  uint64_t y_zero_n;               // 16-byte units
  unsigned long long* grid_bar;    // [count, generation], zero-initialised once per context
};

// Bounded mbarrier waits: a wait that does not complete within ~4 s of clock64 cycles
// prints which barrier stalled and traps (an error on the host instead of a hung GPU).
template <bool kCluster>
APMM_DEV uint32_t mbar_try(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  if (kCluster) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
  }
  return ok;
}
template <bool kCluster = false>
APMM_DEV void mbar_wait_b(uint64_t* bar, uint32_t parity, int what,
                          unsigned long long* acc = nullptr) {
  const uint32_t addr = smem_u32(bar);
  if (mbar_try<kCluster>(addr, parity)) return;
  const long long t0 = clock64();
  struct Acc {
    unsigned long long* a;
    long long t0;
    __device__ ~Acc() { if (a) *a += clock64() - t0; }
  } guard{acc, t0};
  while (!mbar_try<kCluster>(addr, parity)) {
    if (clock64() - t0 > 8000000000ll) {
      printf("[apmm fused] barrier wait timeout: block %d warp %d what %d parity %u\n",
             blockIdx.x, threadIdx.x >> 5, what, parity);
      __trap();
    }
  }
}

APMM_DEV void tma_load_3d_local(uint32_t dst, const void* tmap, uint32_t bar, int32_t c0,
                                int32_t c1, int32_t c2, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(hint)
      : "memory");
}

// Arrive on an mbarrier anywhere in the cluster with the default (.release.cta) semantics.
// The .release.cluster form (ptx.cuh mbar_arrive_cluster) compiles to MEMBAR.ALL.GPU and
// serialised the transform warps (ncu: ERRBAR/MEMBAR top stalls, 137 us at 4096^3); the
// data it publishes is this CTA's own shared memory, already handed to the async proxy by
// fence.proxy.async, so CTA-scope release is what the MMA needs (as CUTLASS's
// ClusterBarrier::arrive(cta_id) does).
APMM_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

APMM_DEV uint2 ld_shared_v2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
APMM_DEV uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// 8x8 bit transpose inside every byte lane (row i = plane i): afterwards byte b of x[c] is
// the code of column 8b + c. Same network as K1's (prep.cu), planes >= NW are zero.
APMM_DEV void swap_sel(uint32_t& a, uint32_t& b, int s, uint32_t m) {
  const uint32_t na = (a & ~(m << s)) | ((b << s) & (m << s));
  b = (b & ~m) | ((a >> s) & m);
  a = na;
}
APMM_DEV void transpose8(uint32_t (&x)[8]) {
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

__device__ __forceinline__ uint32_t dequant_bits(uint32_t v, double sw, double sx) {
  return __float_as_uint(static_cast<float>(__dmul_rn(__dmul_rn(double(int(v)), sw), sx)));
}

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

struct Unit {
  TileInfo ti;
  uint32_t kb0, kb1;
  bool first;  // adds the rank-1 recovery term (the K range starting at 0)
};
__device__ __forceinline__ Unit unit_info(uint32_t u, const Params& p) {
  if (!p.split) return {tile_info(u, p.tiles_m, p.tiles_n, p.n_full), 0u, p.kblocks, true};
  const uint32_t t = u / p.split, ks = u - t * p.split;
  uint32_t tm, tn;
  raster_tile(t, p.tiles_m, p.tiles_n_split, tm, tn);
  const uint32_t kb0 = ks * p.kb_per;
  const uint32_t kb1 = kb0 + p.kb_per < p.kblocks ? kb0 + p.kb_per : p.kblocks;
  return {{tm, tn * p.ncols, p.ncols}, kb0, kb1, ks == 0};
}

// TMA reduce-add of a staged 32x32 int32 tile into Y (split-K partial sums; exact mod 2^32)
APMM_DEV void tma_reduce_add_2d(const void* tmap, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
      : "memory");
}

// NW: planes handled at compile time (1..4 exact; 8 covers 5..8 with runtime masking).
template <int NW>
// Register cap: 384 x 136 leaves room for one K1 block (128 x 80) beside the resident CTA,
// so the next call's K1 overlaps this GEMM (PDL) instead of queueing behind it.
__global__ void __maxnreg__(kXformWarpsCfg == 4 ? 136 : 108)
    gemm_pair_wplanes_kernel(const __grid_constant__ CUtensorMap tmap_wp,
                             const __grid_constant__ CUtensorMap tmap_x,
                             const __grid_constant__ CUtensorMap tmap_x64,
                             const __grid_constant__ CUtensorMap tmap_y, const Params p) {
  constexpr int kStages = op_stages(NW);
  constexpr int kStageBytes = kOpStageBytes;
  constexpr int kRawStages = raw_stages(NW);
  constexpr int kRawBytes = raw_bytes(NW);
  constexpr int kRB = raw_rb(NW);
  constexpr int kRawPlane = raw_plane(NW);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  uint8_t* stages = smem;  // per operand stage: [A codes 16K | B codes 16K]
  uint8_t* raw_ring = smem + kStages * kStageBytes;
  uint8_t* staging = raw_ring + kRawStages * kRawBytes;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + 4 * 2 * kEpiBuf);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* raw_full = empty_bar + kStages;
  uint64_t* raw_empty = raw_full + kRawStages;
  uint64_t* tmem_full = raw_empty + kRawStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  // split mode: rowsum(U_w) of this CTA's 128 rows over the unit's K range, computed by the
  // transform warps (sum_i 2^i popc(plane words)), double-buffered like the accumulators
  __shared__ int32_t rsw_s[2][kHalf];
  __shared__ __align__(8) uint64_t rsw_full[2], rsw_empty[2];
  __shared__ __align__(8) uint64_t x_ready;  // xprep: the grid-wide feature prep is done
  __shared__ __align__(16) uint32_t xterm_s[4][kPairN];  // epilogue: per-warp column terms

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  auto stamp = [&](int k) {
    if (p.ts && !p.ts_clock && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.ts[blockIdx.x * 8 + k] = t;
    }
  };
  stamp(0);
  const uint32_t q = cluster_ctarank() & 1u;  // 0 = MMA leader
  const uint32_t lead_rank = 0;
  const bool leader = q == 0;
  const uint32_t cluster = blockIdx.x / 2;
  const uint32_t nclusters = gridDim.x / 2;
  const uint32_t num_tiles = p.split ? p.tiles_m * p.tiles_n_split * p.split
                                    : p.n_full + 2 * (p.tiles_m * p.tiles_n - p.n_full);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_wp);
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_x64);
    if (p.tma_store) tma_prefetch_desc(&tmap_y);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1 + 2 * kXformWarps);  // leader's expect_tx + transforms
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < kRawStages; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], kXformWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], 8);
      mbar_init(&rsw_full[s], kXformWarps);
      mbar_init(&rsw_empty[s], 4);
    }
    mbar_init(&x_ready, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL. The weight planes are inputs of the call (apmm_cuda.h: readable before the previous
  // kernel completes), so with early_w the raw-plane producer, the transform warps and the
  // MMA issuer start at once: the first operand stages fill while the previous kernel (K1,
  // expanding X) drains. The feature-code producer (K1's output) and the epilogue (rowsum(U_x),
  // Y) wait for it.
  if (!p.early_w || warp == 0 || (warp >= 4 && warp < kXformWarp0)) pdl_wait();
  if (threadIdx.x == 0) pdl_trigger();
  stamp(1);

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (elect_one()) {
      const uint64_t hint = policy_evict_last();
      uint32_t stage = 0, phase = 0;
      if (p.xprep) {  // the feature codes are written by this grid (every CTA's epilogue warps)
        mbar_wait_b(&x_ready, 0, 10);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      for (uint32_t t = cluster; t < num_tiles; t += nclusters) {
        const Unit un = unit_info(t, p);
        const TileInfo ti = un.ti;
        const bool half = ti.ncols != kPairN;
        for (uint32_t kb = un.kb0; kb < un.kb1; ++kb) {
          mbar_wait_b(&empty_bar[stage], phase ^ 1, 1);
          uint8_t* st = stages + stage * kStageBytes;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], (p.ablate & 2) ? 0 : half ? kAS : 2 * kAS);
          if (p.ablate & 2) {
            if (++stage == kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          const uint32_t fb = mapa(smem_u32(&full_bar[stage]), lead_rank);
          if (half) {
            tma_load_2d_pair(st + kAS, &tmap_x64, fb, int32_t(kb * kBK),
                             int32_t(ti.col0 + q * (kHalf / 2)), hint);
          } else {
            tma_load_2d_pair(st + kAS, &tmap_x, fb, int32_t(kb * kBK),
                             int32_t(ti.col0 + q * kHalf), hint);
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
      unsigned long long* af = p.dbg ? &w_full : nullptr;
      unsigned long long* at = p.dbg ? &w_tmem : nullptr;
      for (uint32_t t = cluster; t < num_tiles; t += nclusters) {
        mbar_wait_b(&tmem_empty[acc], acc_phase ^ 1, 2, at);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kPairN;
        const Unit un = unit_info(t, p);
        const uint32_t idesc = un.ti.ncols != kPairN ? kIdescHalf : kIdesc;
        for (uint32_t kb = un.kb0; kb < un.kb1; ++kb) {
          // CTA-scope acquire (as CUTLASS's ClusterBarrier::wait): the stage is read by the
          // tensor core (async proxy); the writers fenced their generic stores to the async
          // proxy before arriving. The cluster-scope form invalidated L1 (CCTL.IVALL) on every
          // poll (ncu source view, profiles/r02_ncu_mid_wplanes.txt).
          mbar_wait_b(&full_bar[stage], phase, 3, af);
          if (p.ts && !p.ts_clock && t == cluster && kb == un.kb0) {  // first operand stage ready
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            p.ts[blockIdx.x * 8 + 2] = tt;
          }
          tc_fence_after();
          const uint32_t st = smem_u32(stages + stage * kStageBytes);
          const uint64_t adesc = umma_desc_sw128(st);
          const uint64_t bdesc = umma_desc_sw128(st + kAS);
#pragma unroll
          for (uint32_t k = 0; k < kBK / 32; ++k) {
            mma_i8_pair(d_tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (kb != un.kb0) || k != 0);
          }
          mma_commit_pair_mc(&empty_bar[stage], 0x3);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        mma_commit_pair_mc(&tmem_full[acc], 0x3);
        if (p.ts && !p.ts_clock) {  // last write = the last unit's MMAs issued
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          p.ts[blockIdx.x * 8 + 3] = tt;
        }
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
  } else if (warp == 3) {
    // ---------------- raw-plane producer (both CTAs): this CTA's 128 weight rows ----------------
    if (elect_one()) {
      const uint64_t hint = policy_evict_last();
      uint32_t rs = 0, rphase = 0;
      for (uint32_t t = cluster; t < num_tiles; t += nclusters) {
        const Unit un = unit_info(t, p);
        const int32_t wrow = int32_t(un.ti.tm * 2 * kHalf + q * kHalf);
        for (uint32_t kb = un.kb0; kb < un.kb1; kb += kRB) {
          mbar_wait_b(&raw_empty[rs], rphase ^ 1, 6);
          mbar_arrive_expect_tx(&raw_full[rs], p.n_w * kRawPlane);
          tma_load_3d_local(smem_u32(raw_ring + rs * kRawBytes), &tmap_wp, smem_u32(&raw_full[rs]),
                            int32_t(kb * (kBK / 32)), wrow, 0, hint);
          if (++rs == kRawStages) { rs = 0; rphase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp >= kXformWarp0) {
    // ---------------- transform: raw planes -> swizzled u8 codes (both CTAs) ----------------
    // thread -> weight row of the tile. A warp's 128-bit plane loads are 512 contiguous
    // bytes (conflict-free); its 128-bit code stores hit 8 distinct 16-B bank groups per
    // quarter warp, because the swizzle XOR spreads consecutive rows. Software pipelined:
    // the codes of K block i+1 are computed while the MMA still reads operand stage i.
    const uint32_t tt = threadIdx.x - kXformWarp0 * 32;
    const uint32_t row = kWPT == 4 ? tt : tt >> 1;       // weight row of the tile
    const uint32_t w0 = kWPT == 4 ? 0u : (tt & 1u) * 2u;  // first of its kWPT words
    const uint32_t sw = row & 7u;
    const uint32_t fb0 = mapa(smem_u32(&full_bar[0]), lead_rank);
    uint32_t stage = 0, phase = 0, rs = 0, rphase = 0;
    uint32_t xa[kWPT][8];
    unsigned long long c_raw = 0;
    uint32_t rsum = 0, rbuf = 0, rphase_e = 0;  // split mode: this unit's rowsum partial
    // the flat sequence of (unit, K block) this CTA's MMA consumes: cursor (fu, fkb) = the
    // block the next fetch() reads, within unit range [fkb0, fkb1)
    uint32_t fu = cluster, fkb0 = 0, fkb1 = 0, fkb = 0;
    auto cursor_load = [&]() {
      if (fu < num_tiles) {
        const Unit un = unit_info(fu, p);
        fkb0 = un.kb0;
        fkb1 = un.kb1;
        fkb = fkb0;
      }
    };
    cursor_load();
    auto cursor_next = [&]() {
      if (++fkb == fkb1) {
        fu += nclusters;
        cursor_load();
      }
    };
    auto fetch = [&](uint32_t kb, uint32_t (&x)[kWPT][8]) {  // raw planes of block kb -> codes
      const uint32_t j = (kb - fkb0) % kRB;  // K block within the raw stage (stages start at kb0)
      if (j == 0) {
        const unsigned long long r0 = p.dbg ? clock64() : 0;
        mbar_wait_b(&raw_full[rs], rphase, 4);
        if (p.dbg) c_raw += clock64() - r0;
      }
      const uint32_t raw = smem_u32(raw_ring + rs * kRawBytes) + row * (16u * kRB) + j * 16u + w0 * 4u;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < NW && (NW <= 4 || uint32_t(i) < p.n_w)) {
          if (kWPT == 4) {
            const uint4 v = ld_shared_v4(raw + i * kRawPlane);
            x[0][i] = v.x;
            x[1 % kWPT][i] = v.y;
            x[2 % kWPT][i] = v.z;
            x[3 % kWPT][i] = v.w;
          } else {
            const uint2 v = ld_shared_v2(raw + i * kRawPlane);
            x[0][i] = v.x;
            x[1][i] = v.y;
          }
        } else {
#pragma unroll
          for (int u = 0; u < kWPT; ++u) x[u][i] = 0u;
        }
      }
      if (kb == fkb0) rsum = 0;
      if (kb * 4u + 3u >= p.last_word) {  // the block holding the row's last plane word
#pragma unroll
        for (int u = 0; u < kWPT; ++u) {
          const uint32_t wd = kb * 4u + w0 + u;
          const uint32_t m = wd < p.last_word ? 0xffffffffu : wd == p.last_word ? p.tail_mask : 0u;
#pragma unroll
          for (int i = 0; i < NW; ++i) x[u][i] &= m;
        }
      }
      if (p.split) {
#pragma unroll
        for (int u = 0; u < kWPT; ++u) {
#pragma unroll
          for (int i = 0; i < NW; ++i) rsum += uint32_t(__popc(x[u][i])) << i;
        }
        if (kb + 1 == fkb1) {  // unit complete: publish the row's partial rowsum
          rsum += __shfl_xor_sync(0xffffffffu, rsum, 1);  // the row's two threads (kWPT = 2)
          mbar_wait_b(&rsw_empty[rbuf], rphase_e ^ 1, 8);
          if (w0 == 0) rsw_s[rbuf][row] = static_cast<int32_t>(rsum);
          __syncwarp();
          if (lane == 0) mbar_arrive(&rsw_full[rbuf]);
          if (++rbuf == 2) { rbuf = 0; rphase_e ^= 1; }
        }
      }
#pragma unroll
      for (int u = 0; u < kWPT; ++u) transpose8(x[u]);
      if (j == kRB - 1 || kb + 1 == fkb1) {
        __syncwarp();  // every lane's plane words are consumed: the slot may be refilled
        if (lane == 0) mbar_arrive(&raw_empty[rs]);
        if (++rs == kRawStages) { rs = 0; rphase ^= 1; }
      }
    };
    unsigned long long c_empty = 0, c_fetch = 0, c_pub = 0;
    const unsigned long long t_loop = clock64();
    bool have = fu < num_tiles;
    if (have) fetch(fkb, xa);
    while (have) {
      const unsigned long long t0 = p.dbg ? clock64() : 0;
      mbar_wait_b(&empty_bar[stage], phase ^ 1, 7);  // the MMA is done with this A slot
      const unsigned long long t1 = p.dbg ? clock64() : 0;
      const uint32_t arow = smem_u32(stages + stage * kStageBytes) + row * 128u;
#pragma unroll
      for (int u = 0; u < kWPT; ++u) {
        if (p.ablate & 1) break;
        const uint32_t c = 2u * (w0 + u);  // word w -> 16-B chunks 2w, 2w+1 of the 128-B row
        st_shared_v4(arow + ((c ^ sw) << 4), xa[u][0], xa[u][1], xa[u][2], xa[u][3]);
        st_shared_v4(arow + (((c + 1u) ^ sw) << 4), xa[u][4], xa[u][5], xa[u][6], xa[u][7]);
      }
      // next block's codes while the stores drain; then publish this stage (a two-block
      // variant with both blocks in flight per iteration measured ~3% slower, r02 notes)
      cursor_next();
      have = fu < num_tiles;
      if (have) fetch(fkb, xa);
      const unsigned long long t2 = p.dbg ? clock64() : 0;
      if (!(p.ablate & 4)) fence_proxy_async_smem();  // generic stores -> async proxy (MMA)
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(fb0 + stage * 8u);
      if (++stage == kStages) { stage = 0; phase ^= 1; }
      if (p.dbg) {
        const unsigned long long t3 = clock64();
        c_empty += t1 - t0;
        c_fetch += t2 - t1;
        c_pub += t3 - t2;
      }
    }
    if (p.dbg && lane == 0) {
      atomicAdd(p.dbg + 4, c_empty);
      atomicAdd(p.dbg + 5, c_fetch);
      atomicAdd(p.dbg + 6, c_pub);
      atomicAdd(p.dbg + 7, clock64() - t_loop);
      atomicAdd(p.dbg + 8, 1ull);
      atomicAdd(p.dbg + 9, c_raw);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs); identical to gemm_pair.cu ----------------
    const uint32_t wq = warp & 3;
    if (p.xprep) {
      // feature prep for the whole grid (rows round-robin over every CTA's 4 epilogue warps),
      // Y zeroed for the reduce-adds, then the grid-wide barrier
      const xpd::ExpandOperand xo{p.x_planes, p.x_codes, p.x_rowsum, p.rows_x, p.rows_x_pad,
                                  static_cast<int>(p.n_x), 0};
      const uint32_t nwarps = gridDim.x * 4u;
      for (uint32_t r = blockIdx.x * 4u + wq; r < p.rows_x; r += nwarps) {
        xpd::expand_one(xo, r, p.wpr, p.tail_mask, p.kpad_words, lane);
      }
      const uint32_t te = wq * 32u + lane;
      if (blockIdx.x == 0) {
        for (uint32_t r = p.rows_x + te; r < p.rows_x_pad; r += 128u) p.x_rowsum[r] = 0;
      }
      for (uint64_t i = uint64_t(blockIdx.x) * 128u + te; i < p.y_zero_n; i += uint64_t(gridDim.x) * 128u) {
        p.y_zero[i] = make_uint4(0, 0, 0, 0);
      }
      // generic-proxy writes -> visible to the async proxy (other CTAs' TMA loads / reduce-adds)
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (wq == 0 && lane == 0) {
        // sense-reversing grid barrier (grid sizes differ between calls): count at
        // grid_bar[0], generation at grid_bar[1]; the last arriver resets the count and
        // advances the generation. A launch starts only after the previous one completed
        // (griddepcontrol.wait above), so barriers of consecutive calls never overlap.
        unsigned long long* count = p.grid_bar;
        unsigned long long* gen = p.grid_bar + 1;
        unsigned long long g0, old;
        asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(g0) : "l"(gen) : "memory");
        asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(count) : "memory");
        if (old + 1 == gridDim.x) {
          asm volatile("st.relaxed.gpu.u64 [%0], 0;" ::"l"(count) : "memory");
          asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(gen), "l"(g0 + 1) : "memory");
        } else {
          unsigned long long now;
          const long long t0 = clock64();
          do {
            asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(now) : "l"(gen) : "memory");
            if (clock64() - t0 > 8000000000ll) {
              printf("[apmm fused] grid barrier timeout: block %d\n", blockIdx.x);
              __trap();
            }
          } while (now == g0);
        }
        mbar_arrive(&x_ready);  // the B producer may load feature codes now
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    uint32_t acc = 0, acc_phase = 0, nbuf = 0;
    const uint64_t store_hint = policy_evict_first();
    for (uint32_t t = cluster; t < num_tiles; t += nclusters) {
      const Unit un = unit_info(t, p);
      const TileInfo ti = un.ti;
      const uint32_t row0 = ti.tm * 2 * kHalf + q * kHalf + wq * 32;
      const uint32_t row = row0 + lane;
      const bool row_ok = row < p.rows_w;
      uint32_t rsw;
      if (p.split) {  // this unit's K-range share of rowsum(U_w), from the transform warps
        mbar_wait_b(&rsw_full[acc], acc_phase, 9);
        rsw = static_cast<uint32_t>(rsw_s[acc][wq * 32 + lane]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&rsw_empty[acc]);
      } else {
        rsw = row_ok ? static_cast<uint32_t>(__ldg(p.rowsum_w + row)) : 0u;
      }
      // split-K: every unit adds its W term (linear in K); the unit holding K block 0 adds
      // the X term and the constant K*A*B once
      const uint32_t row_term = (un.first ? p.c0 : 0u) - p.coef_w * rsw;
      const uint32_t coef_x = un.first ? p.coef_x : 0u;
      double swv = 0.0;
      if (p.yf) swv = p.gran_w ? (row_ok ? p.s_w[row] : 0.0) : p.s_w[0];

      // this unit's column terms coef_x * rowsum(U_x) into the warp's shared row BEFORE
      // waiting for the accumulator; each chunk then reads its 32 terms as 8 broadcast
      // 128-bit loads (a shuffle per column cost ~450 cycles per chunk, dev cycle trace)
      {
        uint4 lo = make_uint4(0, 0, 0, 0), hi = make_uint4(0, 0, 0, 0);
        if (8u * lane < ti.ncols) {
          const int4* src = reinterpret_cast<const int4*>(p.rowsum_x + ti.col0 + 8u * lane);
          // written by this grid's feature prep (xprep): coherent L2 loads, never the
          // read-only path (ld.global.nc may serve data cached before the grid barrier)
          const int4 a = p.xprep ? __ldcg(src) : __ldg(src);
          const int4 b = p.xprep ? __ldcg(src + 1) : __ldg(src + 1);
          lo = make_uint4(coef_x * uint32_t(a.x), coef_x * uint32_t(a.y), coef_x * uint32_t(a.z),
                          coef_x * uint32_t(a.w));
          hi = make_uint4(coef_x * uint32_t(b.x), coef_x * uint32_t(b.y), coef_x * uint32_t(b.z),
                          coef_x * uint32_t(b.w));
        }
        __syncwarp();  // the previous unit's reads of this row are done
        reinterpret_cast<uint4*>(&xterm_s[wq][0])[2 * lane] = lo;
        reinterpret_cast<uint4*>(&xterm_s[wq][0])[2 * lane + 1] = hi;
        __syncwarp();
      }
      mbar_wait_b(&tmem_full[acc], acc_phase, 5);
      tc_fence_after();
      if (p.ts && !p.ts_clock && lane == 0 && warp == 4) {  // accumulator ready (last write = last unit)
        unsigned long long tt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
        p.ts[blockIdx.x * 8 + 6] = tt;
      }
      const uint32_t t_addr = tmem_base + ((wq * 32u) << 16) + acc * kPairN;
      // dev fine trace: cycles of the first two chunks of the CTA's last unit (warp 4, lane 0)
      const bool fine = p.ts && p.ts_clock && lane == 0 && warp == 4 && t + nclusters >= num_tiles;
      long long f0 = fine ? clock64() : 0;
      auto fstamp = [&](int k) {
        if (fine) p.ts[blockIdx.x * 8 + k] = static_cast<unsigned long long>(clock64() - f0);
      };
#pragma unroll 1
      for (uint32_t c = 0; c < ti.ncols / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(t_addr + c * 32, r);
        tmem_ld_wait();
        if (c < 2) fstamp(1 + 3 * c);  // [1] / [4]: accumulator chunk in registers
        const uint32_t col0 = ti.col0 + c * 32;
        const uint4* xt = reinterpret_cast<const uint4*>(&xterm_s[wq][c * 32]);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const uint4 v = xt[j4];  // same address in every lane: one broadcast wavefront
          r[4 * j4 + 0] = 4u * r[4 * j4 + 0] + row_term - v.x;
          r[4 * j4 + 1] = 4u * r[4 * j4 + 1] + row_term - v.y;
          r[4 * j4 + 2] = 4u * r[4 * j4 + 2] + row_term - v.z;
          r[4 * j4 + 3] = 4u * r[4 * j4 + 3] + row_term - v.w;
        }
        if (p.yf) {
          if (p.gran_x) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const uint32_t cj = col0 + j < p.rows_x ? col0 + j : 0;
              r[j] = dequant_bits(r[j], swv, __ldg(p.s_x + cj));
            }
          } else {
            const double sx = p.s_x[0];
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = dequant_bits(r[j], swv, sx);
          }
        }
        if (c < 2) fstamp(2 + 3 * c);  // [2] / [5]: recovery math done
        if (p.tma_store) {
          uint8_t* buf = staging + (wq * 2 + nbuf) * kEpiBuf;
          nbuf ^= 1;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          const uint32_t base = smem_u32(buf) + lane * 128u;
#pragma unroll
          for (uint32_t ch = 0; ch < 8; ++ch) {
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
          if (c < 2) fstamp(3 + 3 * c);  // [3] / [6]: staged, fenced, bulk op issued
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
      fstamp(7);  // [7]: every chunk of the unit issued
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa(smem_u32(&tmem_empty[acc]), lead_rank));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (p.ts && !p.ts_clock && lane == 0 && warp == 4) {  // chunks issued (last write = last unit)
        unsigned long long tt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
        p.ts[blockIdx.x * 8 + 7] = tt;
      }
    }
    // the staging buffers must have been read before the CTA exits; the stores themselves
    // complete with the grid (as CUTLASS's tma_store_wait), so no write round trip here
    if (lane == 0) bulk_wait_read<0>();
    if (p.ts && !p.ts_clock && lane == 0 && warp == 4) {  // epilogue drained
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      p.ts[blockIdx.x * 8 + 5] = tt;
    }
    __syncwarp();
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
  stamp(4);
}

template <int NW>
cudaError_t launch_nw(const CUtensorMap& twp, const CUtensorMap& tx, const CUtensorMap& tx64,
                      const CUtensorMap& ty, Params p, uint32_t full_tiles, int num_sms,
                      cudaStream_t s) {
  auto kern = gemm_pair_wplanes_kernel<NW>;
  static int max_clusters_dev[kMaxDevices] = {};
  int& max_clusters = max_clusters_dev[current_device()];
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes(NW);
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 2;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (!max_clusters) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem_bytes(NW));
    if (e != cudaSuccess) {
      std::fprintf(stderr, "[apmm fused] smem attribute (%d B): %s\n", smem_bytes(NW),
                   cudaGetErrorString(e));
      return e;
    }
    cfg.gridDim = dim3(static_cast<unsigned>(num_sms / 2 * 2));
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    max_clusters = (e == cudaSuccess && n > 0) ? n : num_sms / 2;
    if (APMM_DEV_ENV("APMM_DEBUG_PLAN")) {
      std::fprintf(stderr, "[apmm fused] NW=%d operand stages=%d raw stages=%d smem=%d: %d co-resident pairs\n",
                   NW, op_stages(NW), raw_stages(NW), smem_bytes(NW), max_clusters);
    }
  }
  const uint32_t mc = static_cast<uint32_t>(max_clusters);
  if (p.split) {  // split-K units: (tiles of ncols) x split
    const uint32_t units = p.tiles_m * p.tiles_n_split * p.split;
    cfg.gridDim = dim3(2 * (units < mc ? units : mc));
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, twp, tx, tx64, ty, p);
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  p.n_full = full_tiles;
  if (APMM_DEV_ENV("APMM_NO_TAIL_SPLIT") == nullptr) {
    const uint32_t r = full_tiles % mc;
    if (r != 0 && 2 * r <= mc) p.n_full = full_tiles - r;
  }
  const uint32_t tiles = p.n_full + 2 * (full_tiles - p.n_full);
  cfg.gridDim = dim3(2 * (tiles < mc ? tiles : mc));
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, twp, tx, tx64, ty, p);
  if (e != cudaSuccess) {
    std::fprintf(stderr, "[apmm fused] launch (grid %u, smem %d): %s\n", cfg.gridDim.x,
                 smem_bytes(NW), cudaGetErrorString(e));
    return e;
  }
  return cudaGetLastError();
}

}  // namespace

// Opt-in (APMM_ROUTE_PAIR_WPLANES): measured slower than K1 + K3 on B200 (4096^3 W2A4: 66-68 us vs
// 51 us). The per-tile re-expansion of W (16x at 4096^3) is ALU work the transform warps
// cannot hide: they need ~550 cycles per K block against ~350 cycles of MMA
// (APMM_DEBUG_WAITS breakdown in profiles/r01b_notes.md). Kept, tested bit-exact, for the
// shapes where it could pay (few N tiles, wide K).
bool gemm_wplanes_addressable(const uint32_t* w_planes, uint64_t k) {
  return ((k + 31) / 32) % 4 == 0 && reinterpret_cast<uintptr_t>(w_planes) % 16 == 0;
}

cudaError_t launch_gemm_pair_wplanes(const GemmArgs& a, const uint32_t* w_planes,
                                     cudaStream_t s, int* launches, bool split_k) {
  const uint64_t wpr = (a.k_logical + 31) / 32;
  CUtensorMap twp, tx, tx64, ty;
  {
    const uint64_t dims[3] = {wpr, a.rows_w, static_cast<uint64_t>(a.n_w)};
    const uint64_t strides[2] = {wpr * 4, wpr * 4 * a.rows_w};
    const uint32_t box[3] = {static_cast<uint32_t>(kBK / 32 * raw_rb(a.n_w <= 4 ? a.n_w : 8)),
                             static_cast<uint32_t>(kHalf), static_cast<uint32_t>(a.n_w)};
    const CUresult r = encode_tmap_3d_u32(&twp, w_planes, dims, strides, box);
    if (r != CUDA_SUCCESS) {
      std::fprintf(stderr, "[apmm fused] weight-plane tensor map encode failed (%d)\n", int(r));
      return cudaErrorInvalidValue;
    }
  }
  if (encode_tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.codes_x, a.kpad, a.rows_x, a.kpad,
                     kBK, kHalf) != CUDA_SUCCESS ||
      encode_tmap_2d(&tx64, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, a.codes_x, a.kpad, a.rows_x, a.kpad,
                     kBK, kHalf / 2) != CUDA_SUCCESS) {
    std::fprintf(stderr, "[apmm fused] feature-code tensor map encode failed\n");
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
    ty = tx;  // unused
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
  p.n_w = static_cast<uint32_t>(a.n_w);
  p.last_word = static_cast<uint32_t>(wpr - 1);
  const uint32_t tail = static_cast<uint32_t>(a.k_logical & 31);
  p.tail_mask = tail ? ((1u << tail) - 1u) : 0xffffffffu;
  p.dbg = a.dbg;
  p.ts = a.trace;
  static const bool ts_clock = APMM_DEV_ENV("APMM_TRACE_CLOCK") != nullptr;
  p.ts_clock = ts_clock ? 1u : 0u;
  p.early_w = a.early_w ? 1u : 0u;
  if (a.xprep_planes) {
    p.xprep = 1u;
    p.x_planes = a.xprep_planes;
    p.x_codes = const_cast<uint8_t*>(a.codes_x);
    p.x_rowsum = const_cast<int32_t*>(a.rowsum_x);
    p.rows_x_pad = static_cast<uint32_t>(a.xprep_rows_pad);
    p.n_x = static_cast<uint32_t>(a.n_x);
    p.wpr = static_cast<uint32_t>(wpr);
    p.kpad_words = static_cast<uint32_t>(a.kpad / 32);
    p.y_zero = reinterpret_cast<uint4*>(a.y);
    p.y_zero_n = a.rows_w * a.rows_x * 4 / 16;
    p.grid_bar = a.grid_bar;
  }
  static const uint32_t ablate = [] {
    const char* e = APMM_DEV_ENV("APMM_FUSED_ABLATE");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
  }();
  p.ablate = ablate;
  const uint32_t full_tiles = p.tiles_m * p.tiles_n;
  if (split_k) {
    // mid-size call: tiles of 128 (M_tok <= 128) or 256 feature rows, K split so that the
    // units fill the co-resident pairs (one per TPC: num_sms / 2)
    p.ncols = a.rows_x <= 128 ? 128u : 256u;
    p.tiles_n_split = static_cast<uint32_t>((a.rows_x + p.ncols - 1) / p.ncols);
    const uint32_t tiles = p.tiles_m * p.tiles_n_split;
    const uint32_t pairs = static_cast<uint32_t>(a.num_sms / 2);
    uint32_t sk = pairs / (tiles ? tiles : 1);
    const uint32_t max_s = p.kblocks / 2 > 0 ? p.kblocks / 2 : 1;  // >= 2 K blocks per unit
    sk = sk < 1 ? 1 : (sk > max_s ? max_s : sk);
    p.kb_per = (p.kblocks + sk - 1) / sk;
    p.split = (p.kblocks + p.kb_per - 1) / p.kb_per;  // no empty units
    if (APMM_DEV_ENV("APMM_DEBUG_PLAN")) {
      std::fprintf(stderr, "[apmm fused] split-K: %u tiles of %u cols x %u K splits of %u blocks\n",
                   tiles, p.ncols, p.split, p.kb_per);
    }
  }
  cudaError_t e;
  switch (a.n_w) {
    case 1: e = launch_nw<1>(twp, tx, tx64, ty, p, full_tiles, a.num_sms, s); break;
    case 2: e = launch_nw<2>(twp, tx, tx64, ty, p, full_tiles, a.num_sms, s); break;
    case 3: e = launch_nw<3>(twp, tx, tx64, ty, p, full_tiles, a.num_sms, s); break;
    case 4: e = launch_nw<4>(twp, tx, tx64, ty, p, full_tiles, a.num_sms, s); break;
    default: e = launch_nw<8>(twp, tx, tx64, ty, p, full_tiles, a.num_sms, s); break;
  }
  *launches += 1;
  return e;
}

}  // namespace apmm_b200
