// stream_tc.cu -- K6: the WnAm bipolar-INT GEMM for small and mid token counts (16 <= M_tok
// <= 128 by AUTO): the packed weight planes are streamed from HBM once, expanded to u8 codes in
// registers and written straight into TENSOR MEMORY, where tcgen05.mma reads them as its A
// operand (kind::i8, A from TMEM, B from shared memory). No code byte of W touches shared
// memory or HBM, and the features are read by the tensor core from shared memory instead of
// being re-loaded into registers for every weight tile (the mma.sync kernel K5 spends most of
// its shared-memory bandwidth on those feature fragments once M_tok > 8).
//
// The algebra is the one of every route (reference kernel.cpp:187-254):
//   Y = 4 * sum_k u_w u_x - 2B * rowsum(U_w) - 2A * rowsum(U_x) + K*A*B   (mod 2^32).
// rowsum(U_w) comes out of the MMA: the feature operand carries an all-ones token row (column
// M_tok of D). Both K-linear terms are formed per K segment, the X term and the constant by the
// segment that holds K step 0, so K may be split anywhere.
//
// Work: the output is cut into tiles of 128 weight rows (the UMMA M) and K into steps of 512
// columns; the tile-steps (tile-major) are dealt to one persistent CTA per SM as contiguous
// ranges (stream-K). A CTA's run of steps of one tile accumulates in TMEM; at its end the
// partial tile is TMA reduce-added (exact wrapping u32 add) into Y, which the feature-prep
// launch (stream_tc_prep_kernel, the call's first launch) zeroed.
//
// CTA: 16 transform warps + 1 MMA warp. Transform warp (q = warp % 4, h = warp / 4) owns the
// 16-row group rg = 2q + (h & 1) of the tile (TMEM lanes 16 rg.., inside its lane quarter q)
// and the CTA's steps of parity h / 2, each written into that parity's 128-column A buffer.
// Per step a warp streams K5's item -- TMA box {16 words, 16 rows, n_w planes}, 64-byte rows,
// conflict-free 16-byte reads with thread (g, t) on words 4t.. of rows g and g + 8 -- through
// its one-slot ring, copies it to registers (the slot is re-issued at once), turns each
// 32-column word into 8 registers of u8 codes with K5's transposes and stores them with
// tcgen05.st.16x256b; the features are written by the prep in the matching permuted K order.
// The MMA warp streams the feature tile of the step (128B swizzle, up to 6 stages) and issues
// 16 MMAs of K = 32 per step. Measured limits: an M=128, K=32 i8 MMA costs
// >= 56 cycles with A in TMEM for N <= 64 (A-operand read, scripts/mma_rate_probe.cu).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace apmm_b200 {
namespace {

using namespace apmm_ptx;

constexpr int kGroups = 2;                      // warp sets: the CTA's even / odd steps
#ifndef APMM_TC_BUFS_AB
constexpr int kBufs = 2;                        // A buffers in TMEM (step i -> buffer i % kBufs)
#else
constexpr int kBufs = APMM_TC_BUFS_AB;          // A/B builds only
#endif
constexpr int kTfWarps = 16;                    // 8 row groups of 16 rows x kGroups sets
constexpr int kMmaWarp = kTfWarps;
constexpr int kThreads = (kTfWarps + 1) * 32;
constexpr uint32_t kStepWords = 16;             // plane words per step (512 columns)
constexpr uint32_t kStepBytes = kStepWords * 32;  // feature code bytes per step and token
constexpr uint32_t kAcols = kStepWords * 8;     // TMEM columns of one A buffer (4 codes each)
constexpr uint32_t kRowBytes = kStepWords * 4;  // bytes of one weight row of one plane per step
constexpr uint32_t kItemRows = 16;              // weight rows per warp item
constexpr int kEpiWarps = 8;                    // warps with an epilogue staging buffer
// Weight ring slots per warp. Deeper rings measured slower (8192 x 16 x 8192 W3A8: 15.2 /
// 15.8 / 18.6 / 18.6 us at 1 / 2 / 3 / 4 slots, profiles/r02/r2_k6_wst.txt; 8192 x 32: 15.9 vs
// 18.3 us at 1 vs 2, r2_k6_ab.txt): the item is copied to registers at once, so one slot
// already overlaps the next item's load with this one's transform.
#ifndef APMM_TC_WST_AB
constexpr uint32_t kMaxWst = 1;
#else
constexpr uint32_t kMaxWst = APMM_TC_WST_AB;  // A/B builds only
#endif
#if defined(APMM_DEVTOOLS) && defined(APMM_TC_DEV_ABLATE)
constexpr bool kDevAblate = true;
#else
constexpr bool kDevAblate = false;
#endif
constexpr uint32_t kTileRows = 128;
#ifndef APMM_TC_BST_AB
// feature-code tiles in flight: up to 6 as shared memory allows (3 at 64 rows, 2 above 80);
// 8192 x 16 x 8192 W3A8 14.95 -> 14.53 us at 6 vs 3 (profiles/r02/r2_k6_bst.txt)
constexpr uint32_t kBStages = 6;
#else
constexpr uint32_t kBStages = APMM_TC_BST_AB;   // A/B builds only
#endif
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColD = kBufs * kAcols;     // A buffers at columns 0 and 128; D from 256
constexpr uint32_t kStageBytes = 32u * 128u;    // per-warp epilogue staging: 32 rows x 32 int32
constexpr uint32_t kSmemCap = 232448u - 2048u;  // opt-in maximum minus static + alignment
constexpr uint32_t kMaxRowsX = 128;
constexpr uint32_t kPrepThreads = 256;

__host__ __device__ constexpr uint32_t n_mma_of(uint32_t rows_x) {
  return rows_x + 1 <= 16 ? 16u : (rows_x + 1 + 15) / 16 * 16;  // + the all-ones token row
}
// Per-warp weight item: 16 rows x 16 words x n planes (one step). PW ("pair" layout): the two
// warps of a row group (one per step parity) share one TMA box of 16 rows x 32 words x n planes
// covering a step pair -- 128-byte row segments instead of 64: K6's stream pattern alone runs
// 25.2 MB in 3.9 instead of 5.9 us (scripts/k6_stream_probe.cu, profiles/r02/r2_k6_stream_probe.txt)
__host__ __device__ constexpr uint32_t wslot_bytes(int n) { return kItemRows * kRowBytes * static_cast<uint32_t>(n); }
__host__ __device__ constexpr uint32_t pslot_bytes(int n) { return 2u * wslot_bytes(n); }
constexpr uint32_t kPairSlots = 2;  // pair boxes in flight per row group
__host__ __device__ constexpr uint32_t b_stage_bytes(uint32_t n_mma) { return n_mma * kStepBytes; }

struct TcParams {
  const int32_t* rsx_part;   // feature prep: rowsum(U_x) parts [n_mma][parts]
  uint32_t parts;
  uint32_t rows_x, n_mma;
  uint32_t n_w;
  uint32_t steps_per_tile;   // K steps per tile
  uint32_t q_steps, r_steps;  // total tile-steps = q * grid + r (CTA c gets q + (c < r))
  uint64_t inv_spt;           // ceil(2^32 / steps_per_tile)
  uint32_t wst;               // per-warp weight ring slots (1..kMaxWst)
  uint32_t bst;               // feature-code ring stages (2..kBStages)
  uint32_t w_off, st_off;     // shared-memory carve-up: B ring at 0, W rings, staging
  uint32_t coef_w, coef_x, c0;
  uint32_t early_w;
  unsigned long long* ts;     // dev builds: per-CTA globaltimer stamps [grid][8], else null
  uint32_t ts_mode;           // dev: 0 phases, 1 MMA warp: step i ready (slot i + 1), 2 warp 0:
                              // its item u landed (slot u + 1), 3 warp 0: item u stored
  uint32_t ablate;            // dev only (APMM_TC_ABLATE, results wrong): 1 no MMAs, 2 no transposes
  uint32_t nd, dstride;       // D accumulators (1 or 2, alternating per segment), columns apart
};

#ifdef APMM_DEVTOOLS
APMM_DEV unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TC_STAMP(ts, slot, k) \
  do {                        \
    if (ts) (ts)[(slot) * 8 + (k)] = gtime_ns(); \
  } while (0)
// ts_mode 5: per-step clock64 events of one CTA in 4 pages of 8 (slot blockIdx.x + 256 page)
#define TC_CLK(pg, k)                                                                       \
  do {                                                                                      \
    if (p.ts && p.ts_mode == 5)                                                             \
      p.ts[(blockIdx.x + 256u * (pg)) * 8u + (k)] = static_cast<unsigned long long>(clock64()); \
  } while (0)
#else
#define TC_CLK(pg, k) \
  do {                \
  } while (0)
#define TC_STAMP(ts, slot, k) \
  do {                        \
  } while (0)
#endif

// floor(n / d) for n, d < 2^16 from inv = ceil(2^32 / d)
APMM_DEV uint32_t div_small(uint32_t n, uint64_t inv) {
  return static_cast<uint32_t>((static_cast<uint64_t>(n) * inv) >> 32);
}

template <uint32_t M>
APMM_DEV uint32_t sel(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(r) : "r"(a), "r"(b), "n"(M));
  return r;
}
// delta swap with both shifts on the FMA pipe (IMAD / IMAD.HI), the selects as LOP3
template <int S>
APMM_DEV void swap_sel(uint32_t& a, uint32_t& b) {
  const uint32_t bs = b * (1u << S);
  const uint32_t as = __umulhi(a, 1u << (32 - S));
  const uint32_t na = S == 1 ? sel<0xAAAAAAAAu>(a, bs) : S == 2 ? sel<0xCCCCCCCCu>(a, bs)
                                                               : sel<0xF0F0F0F0u>(a, bs);
  b = S == 1 ? sel<0x55555555u>(b, as) : S == 2 ? sel<0x33333333u>(b, as) : sel<0x0F0F0F0Fu>(b, as);
  a = na;
}

// u8 codes of one 32-column word (x[i] = plane i's word, zero for i >= N): o[r] byte b = code
// of column 8b + r. N <= 4: two swap stages leave nibble pairs (column 8b+r low, 8b+4+r high).
template <int N>
APMM_DEV void codes_of_word(uint32_t (&x)[8], uint32_t* o) {
  if (N <= 4) {
    swap_sel<2>(x[0], x[2]);
    swap_sel<2>(x[1], x[3]);
    swap_sel<1>(x[0], x[1]);
    swap_sel<1>(x[2], x[3]);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      o[r] = x[r] & 0x0F0F0F0Fu;
      o[4 + r] = __umulhi(x[r], 1u << 28) & 0x0F0F0F0Fu;  // x >> 4 on the FMA pipe
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) swap_sel<4>(x[i], x[i + 4]);
#pragma unroll
    for (int i = 0; i < 8; i += 4) {
      swap_sel<2>(x[i], x[i + 2]);
      swap_sel<2>(x[i + 1], x[i + 3]);
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2) swap_sel<1>(x[i], x[i + 1]);
#pragma unroll
    for (int r = 0; r < 8; ++r) o[r] = x[r];
  }
}

APMM_DEV void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar, int32_t c0, int32_t c1,
                          int32_t c2, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(hint)
      : "memory");
}
APMM_DEV void tma_reduce_add_2d(const void* tmap, const void* smem_src, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(smem_u32(smem_src)), "r"(c0), "r"(c1)
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem]^T (kind::i8, u8 x u8 -> s32)
APMM_DEV void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
APMM_DEV void tmem_st_16x256b_x8(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
APMM_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
APMM_DEV uint32_t tmem_ld_32x32b_x1(uint32_t taddr) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
  return v;
}

template <int N, bool PW>
__global__ void __launch_bounds__(kThreads, 1)
    stream_tc_kernel(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x,
                     const __grid_constant__ CUtensorMap tm_y, const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t wfull[kTfWarps * kMaxWst];
  __shared__ __align__(8) uint64_t wempty[8 * kPairSlots];  // PW: both warps of the row group read it
  __shared__ __align__(8) uint64_t bfull[kBStages], bempty[kBStages];
  __shared__ __align__(8) uint64_t afull[kBufs], aempty[kBufs], dfull[2], dempty[2];
  __shared__ uint32_t tmem_base_s;
  __shared__ int32_t rsx_s[kMaxRowsX];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) TC_STAMP(p.ts, blockIdx.x, 0);
  if (tid == 0) TC_CLK(3, 0);
  if (tid == 32) {  // descriptor fetches off the first loads (warp 0 initialises the barriers)
    tma_prefetch_desc(&tm_w);
    tma_prefetch_desc(&tm_x);
    tma_prefetch_desc(&tm_y);
  }
  // this CTA's tile-steps [a, b) (PW: q / r count step pairs)
  constexpr uint32_t unit = PW ? 2u : 1u;
  const uint32_t a = unit * (blockIdx.x * p.q_steps + min(blockIdx.x, p.r_steps));
  const uint32_t n_steps = unit * (p.q_steps + (blockIdx.x < p.r_steps ? 1u : 0u));
  const uint32_t b = a + n_steps;
  const uint32_t spt = p.steps_per_tile;

  if (tid == 0) {
    for (int i = 0; i < kTfWarps * kMaxWst; ++i) mbar_init(&wfull[i], 1);
    for (uint32_t i = 0; i < 8 * kPairSlots; ++i) mbar_init(&wempty[i], 2);
    for (uint32_t i = 0; i < kBStages; ++i) {
      mbar_init(&bfull[i], 1);
      mbar_init(&bempty[i], 1);
    }
    for (int i = 0; i < kBufs; ++i) {
      mbar_init(&afull[i], kTfWarps / kGroups);  // one arrive per warp filling the buffer
      mbar_init(&aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dfull[i], 1);
      mbar_init(&dempty[i], kTfWarps);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    TC_CLK(3, 2);
  }
  if (warp == kMmaWarp) tmem_alloc<kTmemCols>(&tmem_base_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) TC_CLK(3, 3);
  const uint32_t tmem = tmem_base_s;
  const uint32_t sbase = smem_u32(smem);

  if (warp < kTfWarps) {
    // ---------------- transform warps ----------------
    // warp (q = warp % 4, h = warp / 4): TMEM lane quarter q, row group rg = 2q + (h & 1) of the
    // tile (16 rows = lanes 16 rg ..), A buffer wg = h / 2 (the CTA's steps of that parity)
    const uint32_t q = warp & 3, h = warp >> 2;
    const uint32_t rg = 2u * q + (h & 1u), wg = h >> 1;
    const uint32_t g = lane >> 2, t = lane & 3;
    // PW: the row group's pair slots (issued by its even-step warp), else this warp's own ring
    const uint32_t wslot0 = sbase + p.w_off + (PW ? rg * kPairSlots * pslot_bytes(N) : warp * p.wst * wslot_bytes(N));
    uint64_t* wbar = wfull + (PW ? rg * kPairSlots : warp * kMaxWst);
    uint64_t* webar = wempty + rg * kPairSlots;
    const bool producer = !PW || wg == 0u;
    const uint64_t hint = policy_evict_first();  // weights are read exactly once
    // this warp's items: steps a + wg, a + wg + kGroups, ...
    uint32_t is_j = a + wg, is_slot = 0;
    auto issue = [&]() {
      if (PW) return;
      if (is_j < b && lane == 0) {
        const uint32_t tile = div_small(is_j, p.inv_spt), s = is_j - tile * spt;
        mbar_arrive_expect_tx(&wbar[is_slot], wslot_bytes(N));
        tma_load_3d(wslot0 + is_slot * wslot_bytes(N), &tm_w, smem_u32(&wbar[is_slot]),
                    int32_t(s * kStepWords), int32_t(tile * kTileRows + rg * kItemRows), 0, hint);
      }
      is_j += kGroups;
      if (++is_slot == p.wst) is_slot = 0;
    };
    // PW: pair k = CTA steps (2k, 2k + 1), one box {32 words, 16 rows, n} into slot k % 2
    auto issue_pair = [&](uint32_t k) {
      if (PW && producer && lane == 0 && 2u * k < n_steps) {
        const uint32_t j = a + 2u * k;
        const uint32_t tile = div_small(j, p.inv_spt), s = j - tile * spt;
        const uint32_t sl = k % kPairSlots;
        mbar_arrive_expect_tx(&wbar[sl], pslot_bytes(N));
        tma_load_3d(wslot0 + sl * pslot_bytes(N), &tm_w, smem_u32(&wbar[sl]),
                    int32_t(s * kStepWords), int32_t(tile * kTileRows + rg * kItemRows), 0, hint);
      }
    };
    if (!p.early_w) pdl_wait();
    if (PW) {
      for (uint32_t k = 0; k < kPairSlots; ++k) issue_pair(k);
    } else {
      for (uint32_t i = 0; i < p.wst; ++i) issue();
    }
    if (tid == 0) TC_CLK(3, 4);
    // The transform warps touch only the weight planes (call inputs), tensor memory and shared
    // memory until their first epilogue: they expand the first steps while the feature prep
    // still runs; griddepcontrol.wait (features' rowsum, Y) comes at the first segment end.
    // rowsum(U_x) is needed only by the first epilogue: loaded there, off the path to the
    // first MMA
    uint8_t* stage = smem + p.st_off + (warp % kEpiWarps) * kStageBytes;
    const uint32_t my_lane_addr = (q * 32u) << 16;          // epilogue: 32x32b over the quarter
    const uint32_t st_lane_addr = (rg * kItemRows) << 16;   // transform: 16x256b, 16 lanes
    uint32_t cs_slot = 0, wphase = 0, uses = 0, segs = 0;
    uint32_t bi = 0, ui = 0;  // step j - a = 3 ui + bi: A buffer bi, its use ui
    uint32_t seg_first_s = 0;  // K step at which the current segment started
    // ---------------- segment epilogue: partial tile -> reduce-add into Y ----------------
    // first: the segment holds K step 0 (X term + constant)
    uint32_t pend_tile = ~0u;
    bool pend_first = false;
    auto epilogue = [&](uint32_t tile, bool first) {
      if (segs == 0) {
        pdl_wait();  // rowsum(U_x) parts and Y only after the prep launch completed
        if (tid == 0 && p.ts_mode == 0) TC_STAMP(p.ts, blockIdx.x, 1);
        if (warp == 0) {
          for (uint32_t c = lane; c < p.rows_x; c += 32) {
            int32_t sum = 0;
            for (uint32_t i = 0; i < p.parts; ++i) sum += __ldg(p.rsx_part + c * p.parts + i);
            rsx_s[c] = sum;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kTfWarps * 32));  // rsx_s visible to the transform warps
      }
      const uint32_t db = p.nd == 2 ? (segs & 1u) : 0u;  // this segment's D buffer
      mbar_wait(&dfull[db], (p.nd == 2 ? segs >> 1 : segs) & 1u);
      tc_fence_after();
      if (tid == 0 && segs == 0) TC_CLK(3, 1);
      if (tid == 0 && segs == 0 && p.ts_mode == 0) TC_STAMP(p.ts, blockIdx.x, 6);
      const uint32_t dcol = tmem + my_lane_addr + kColD + db * p.dstride;
      const uint32_t rsw = tmem_ld_32x32b_x1(dcol + p.rows_x);
      tmem_ld_wait();
      const uint32_t chunks = (p.rows_x + 31) / 32;
      for (uint32_t cc = h; cc < chunks && warp < kEpiWarps; cc += 2) {
        uint32_t d[32];
        tmem_ld_32x32b_x32(dcol + cc * 32u, d);
        tmem_ld_wait();
        if (lane == 0) bulk_wait_read<0>();  // the staging buffer's previous reduce-add read it
        __syncwarp();
  #pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          uint32_t v[4];
  #pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t col = cc * 32u + c4 * 4u + e;
            uint32_t t = 4u * d[c4 * 4 + e] - p.coef_w * rsw;
            if (first && col < p.rows_x) t += p.c0 - p.coef_x * static_cast<uint32_t>(rsx_s[col]);
            v[e] = t;
          }
          st_shared_v4(smem_u32(stage) + lane * 128u + ((c4 ^ (lane & 7u)) << 4), v[0], v[1], v[2], v[3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_reduce_add_2d(&tm_y, stage, int32_t(cc * 32u), int32_t(tile * kTileRows + q * 32u));
          bulk_commit();
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[db]);
      ++segs;
    };
    for (uint32_t j = a; j < b; ++j) {
      const uint32_t tile = div_small(j, p.inv_spt), s = j - tile * spt;
      if (j == a || s == 0) seg_first_s = s;
      if (((j - a) & (kGroups - 1u)) == wg) {
        // the MMAs that read this A buffer three steps ago (the other warp set's) are done
        if (ui > 0) mbar_wait(&aempty[bi], (ui - 1) & 1u);
        const uint32_t si = j - a;  // this CTA's step index
        if ((warp == 0 || warp == 8) && lane == 0 && si < 4) TC_CLK(0, si);
        if (tid == 0 && uses == 1 && p.ts_mode == 4) TC_STAMP(p.ts, blockIdx.x, 6);
        tc_fence_after();
        const uint32_t pk = si >> 1;  // PW: this step's pair
        if (PW) {
          mbar_wait(&wbar[pk % kPairSlots], (pk / kPairSlots) & 1u);
        } else {
          mbar_wait(&wbar[cs_slot], (wphase >> cs_slot) & 1u);
          wphase ^= 1u << cs_slot;
        }
        if ((warp == 0 || warp == 8) && lane == 0 && si < 4) TC_CLK(0, 4 + si);
        if (tid == 0 && uses == 0 && p.ts_mode == 0) TC_STAMP(p.ts, blockIdx.x, 2);
        if (tid == 0 && uses < 6 && p.ts_mode == 2) TC_STAMP(p.ts, blockIdx.x, uses + 1);
        // slot layout (TMA box {16 words, 16 rows, planes}): [plane][row][16 words]; thread
        // (g, t) takes words 4t..4t+3 of rows g and g + 8 (conflict-free 16-byte reads)
        uint4 wa[N], wb[N];
        // PW slot: [plane][16 rows][32 words] (128-byte rows), this warp's half = its step's
        // 16 words; else [plane][16 rows][16 words]
        constexpr uint32_t rbytes = PW ? 2u * kRowBytes : kRowBytes;
        const uint32_t rowb = (PW ? wslot0 + (pk % kPairSlots) * pslot_bytes(N) + wg * kRowBytes
                                  : wslot0 + cs_slot * wslot_bytes(N)) + g * rbytes + t * 16u;
#pragma unroll
        for (int pl = 0; pl < N; ++pl) {
          const uint32_t addr = rowb + pl * kItemRows * rbytes;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(wa[pl].x), "=r"(wa[pl].y), "=r"(wa[pl].z), "=r"(wa[pl].w) : "r"(addr));
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(wb[pl].x), "=r"(wb[pl].y), "=r"(wb[pl].z), "=r"(wb[pl].w)
                       : "r"(addr + 8u * rbytes));
        }
        __syncwarp();
        if (PW) {
          if (lane == 0) mbar_arrive(&webar[pk % kPairSlots]);
          // the even-step warp refills the previous pair's slot (both halves read) with pair pk + 1
          if (producer && pk >= 1) {
            if (lane == 0) mbar_wait(&webar[(pk - 1) % kPairSlots], ((pk - 1) / kPairSlots) & 1u);
            issue_pair(pk + 1);
          }
          __syncwarp();
        } else {
          if (++cs_slot == p.wst) cs_slot = 0;
          issue();  // the slot is free again: the item after next of this warp
        }
        // tcgen05.st.16x256b: register 4jj + e of thread (g, t) -> lane g + 8 (e >> 1), column
        // 8jj + 2t + (e & 1) (profiles/r02/r2_tmem_layout.txt). Word 4t + w of the step, code
        // register r -> column 32 w + 8 (r >> 1) + 2t + (r & 1): the feature prep writes X in the
        // same permuted K order (stream_tc_prep_kernel).
        const uint32_t acol = tmem + st_lane_addr + bi * kAcols;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          uint32_t oa[2][8], ob[2][8];
#pragma unroll
          for (int w2 = 0; w2 < 2; ++w2) {
            const int wd = half * 2 + w2;
            uint32_t xa[8], xb[8];
#pragma unroll
            for (int pl = 0; pl < 8; ++pl) {
              const uint4& va = wa[pl < N ? pl : 0];
              const uint4& vb = wb[pl < N ? pl : 0];
              xa[pl] = pl < N ? (wd == 0 ? va.x : wd == 1 ? va.y : wd == 2 ? va.z : va.w) : 0u;
              xb[pl] = pl < N ? (wd == 0 ? vb.x : wd == 1 ? vb.y : wd == 2 ? vb.z : vb.w) : 0u;
            }
            if (kDevAblate && (p.ablate & 2u)) {
#pragma unroll
              for (int r = 0; r < 8; ++r) {
                oa[w2][r] = xa[r & (N - 1)];
                ob[w2][r] = xb[r & (N - 1)];
              }
            } else {
              codes_of_word<N>(xa, oa[w2]);
              codes_of_word<N>(xb, ob[w2]);
            }
          }
          uint32_t o[32];
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int w2 = jj >> 2, r0 = 2 * (jj & 3);
            o[4 * jj + 0] = oa[w2][r0];
            o[4 * jj + 1] = oa[w2][r0 + 1];
            o[4 * jj + 2] = ob[w2][r0];
            o[4 * jj + 3] = ob[w2][r0 + 1];
          }
          tmem_st_16x256b_x8(acol + half * 64u, o);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[bi]);
        if ((warp == 0 || warp == 8) && lane == 0 && j - a < 4) TC_CLK(1, j - a);
        if (tid == 0 && uses == 0 && p.ts_mode == 0) TC_STAMP(p.ts, blockIdx.x, 3);
        if (tid == 0 && uses < 6 && p.ts_mode == 3) TC_STAMP(p.ts, blockIdx.x, uses + 1);
        ++uses;
      }
      if (++bi == kBufs) {
        bi = 0;
        ++ui;
      }
      if (s + 1 == spt || j + 1 == b) {
        // segment end: with two D buffers the epilogue of a segment runs at the end of the
        // next one (its MMAs drain meanwhile and the transform warps go on to the next
        // segment's steps), else at once
        if (p.nd == 2) {
          if (pend_tile != ~0u) epilogue(pend_tile, pend_first);
          pend_tile = tile;
          pend_first = seg_first_s == 0;
        } else {
          epilogue(tile, seg_first_s == 0);
        }
      }
    }
    if (pend_tile != ~0u) epilogue(pend_tile, pend_first);
    if (lane == 0) bulk_wait<0>();
  } else {
    // ---------------- MMA warp: feature tiles + tcgen05.mma ----------------
    if (lane == 0) {
      const uint32_t idesc = idesc_i8_u8u8(kTileRows, p.n_mma);
      const uint64_t hint = policy_evict_last();  // the feature codes are re-read by every CTA
      const uint32_t bst = p.bst;
      auto load_b = [&](uint32_t i) {  // feature codes of step a + i into stage i % bst
        const uint32_t j = a + i;
        const uint32_t tile = div_small(j, p.inv_spt), s = j - tile * spt;
        const uint32_t st = i % bst;
        uint8_t* dst = smem + st * b_stage_bytes(p.n_mma);
        mbar_arrive_expect_tx(&bfull[st], b_stage_bytes(p.n_mma));
#pragma unroll
        for (int kg = 0; kg < int(kStepBytes / 128); ++kg)
          tma_load_2d(dst + kg * p.n_mma * 128u, &tm_x, &bfull[st], int32_t(s * kStepBytes + kg * 128u), 0, hint);
      };
      pdl_wait();  // the feature codes are written by the prep launch right before us
      for (uint32_t i = 0; i < bst && i < n_steps; ++i) load_b(i);
      uint32_t segs = 0;
      bool seg_open = false;
      for (uint32_t i = 0; i < n_steps; ++i) {
        const uint32_t j = a + i, ab = i % kBufs;
        const uint32_t tile = div_small(j, p.inv_spt), s = j - tile * spt;
        const uint32_t st = i % bst;
        mbar_wait(&bfull[st], (i / bst) & 1u);
        mbar_wait(&afull[ab], (i / kBufs) & 1u);
        const uint32_t db = p.nd == 2 ? (segs & 1u) : 0u, ds = p.nd == 2 ? segs >> 1 : segs;
        if (!seg_open && ds > 0) mbar_wait(&dempty[db], (ds - 1) & 1u);  // epilogue read this D
        tc_fence_after();
        const uint32_t bstage = sbase + st * b_stage_bytes(p.n_mma);
        if (i < 4) TC_CLK(1, 4 + i);
        if (i < 3 && p.ts_mode == 4) TC_STAMP(p.ts, blockIdx.x, 2 * i + 1);
#pragma unroll
        for (uint32_t k = 0; k < ((kDevAblate && (p.ablate & 1u)) ? 1u : kStepBytes / 32); ++k) {
          const uint64_t bdesc = umma_desc_sw128(bstage + (k >> 2) * p.n_mma * 128u + (k & 3u) * 32u);
          mma_i8_ts(tmem + kColD + db * p.dstride, tmem + ab * kAcols + k * 8u, bdesc, idesc, (seg_open || k > 0) ? 1u : 0u);
        }
        seg_open = true;
        if (i < 4) TC_CLK(2, i);
        if (i < 2 && p.ts_mode == 4) TC_STAMP(p.ts, blockIdx.x, 2 * i + 2);
        if (i == 0 && p.ts_mode == 0) TC_STAMP(p.ts, blockIdx.x, 4);
        if (i + 1 == n_steps && p.ts_mode == 0) TC_STAMP(p.ts, blockIdx.x, 5);
        if (i < 6 && p.ts_mode == 1) TC_STAMP(p.ts, blockIdx.x, i + 1);
        mma_commit(&aempty[ab]);
        mma_commit(&bempty[st]);
        if (s + 1 == spt || j + 1 == b) {
          mma_commit(&dfull[db]);
          seg_open = false;
          ++segs;
        }
        // refill the stage of step i - 1 (its MMAs were issued a step ago) with step i + 2
        if (i >= 1 && i + bst - 1 < n_steps) {
          const uint32_t pst = (i - 1) % bst;
          mbar_wait(&bempty[pst], ((i - 1) / bst) & 1u);
          if (i < 4) TC_CLK(2, 4 + i);
          load_b(i + bst - 1);
        }
      }
    }
    __syncwarp();
  }
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) TC_STAMP(p.ts, blockIdx.x, 7);
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem);
  }
}

// Feature prep: X planes -> u8 codes [n_mma][kpad] in the K1 order (rows >= rows_x: the
// all-ones row at rows_x, zeros after), rowsum(U_x) parts, and Y zeroed for the reduce-adds.
// thread = (code row, 32-column word). PDL: triggers at once; reads X and writes its outputs
// only after griddepcontrol.wait (X may be the previous kernel's output, and the previous
// call's GEMM may still read the codes) unless early_x.
__global__ void __launch_bounds__(kPrepThreads) stream_tc_prep_kernel(
    const uint32_t* __restrict__ x, uint32_t rows_x, uint32_t x_rows, uint32_t wpr, int n_x, uint32_t kwords,
    uint8_t* __restrict__ codes, int32_t* __restrict__ rsx_part, uint4* __restrict__ y_zero,
    uint64_t y_vec4, uint32_t early_x, unsigned long long* ts) {
  const uint32_t bslot = blockIdx.y * gridDim.x + blockIdx.x;
  if (threadIdx.x == 0 && bslot < 1024) TC_STAMP(ts, bslot, 0);
  pdl_trigger();
  if (!early_x) pdl_wait();
  if (threadIdx.x == 0 && bslot < 1024) TC_STAMP(ts, bslot, 1);
  const uint32_t row = blockIdx.y, W = blockIdx.x * kPrepThreads + threadIdx.x;
  uint32_t v[8];
  int32_t rs = 0;
  // rows_x: the (4-aligned) code rows before the all-ones row; x_rows <= rows_x of them are X's
  const bool real = row < x_rows;
  const uint64_t pstride = uint64_t(x_rows) * wpr;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = (real && i < n_x && W < wpr) ? __ldg(x + i * pstride + uint64_t(row) * wpr + W) : 0u;
    rs += __popc(v[i]) << i;
  }
  if (early_x) pdl_wait();
  if (real) {
    // 8x8 transpose in all four byte lanes: register r, byte b <- column 8b + r
    auto sw = [](uint32_t& a, uint32_t& b, int s, uint32_t m) {
      const uint32_t na = (a & ~(m << s)) | ((b << s) & (m << s));
      b = (b & ~m) | ((a >> s) & m);
      a = na;
    };
#pragma unroll
    for (int i = 0; i < 4; ++i) sw(v[i], v[i + 4], 4, 0x0F0F0F0Fu);
#pragma unroll
    for (int i = 0; i < 8; i += 4) {
      sw(v[i], v[i + 2], 2, 0x33333333u);
      sw(v[i + 1], v[i + 3], 2, 0x33333333u);
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2) sw(v[i], v[i + 1], 1, 0x55555555u);
  } else {
    const uint32_t c = row == rows_x ? 0x01010101u : 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = c;
  }
  if (W < kwords) {
    // K order of the A operand (see the transform warps): within a 512-column step, word
    // 4t + w, code register r -> 32-bit column 32 w + 8 (r >> 1) + 2t + (r & 1)
    const uint32_t wl = W % kStepWords, t = wl >> 2, w = wl & 3u;
    uint32_t* dst = reinterpret_cast<uint32_t*>(codes + uint64_t(row) * kwords * 32u +
                                                uint64_t(W / kStepWords) * kStepBytes) +
                    32u * w + 2u * t;
#pragma unroll
    for (int r = 0; r < 8; r += 2)
      *reinterpret_cast<uint2*>(dst + 8 * (r >> 1)) = make_uint2(v[r], v[r + 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
  __shared__ int32_t part[kPrepThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = rs;
  __syncthreads();
  if (threadIdx.x == 0 && row < rows_x) {  // (padding rows: zero codes, zero rowsum)
    int32_t s = 0;
    for (int i = 0; i < kPrepThreads / 32; ++i) s += part[i];
    rsx_part[uint64_t(row) * gridDim.x + blockIdx.x] = s;
  }
  // zero Y (grid-stride over the whole launch)
  const uint64_t nthreads = uint64_t(gridDim.x) * gridDim.y * kPrepThreads;
  const uint64_t gtid = (uint64_t(blockIdx.y) * gridDim.x + blockIdx.x) * kPrepThreads + threadIdx.x;
  for (uint64_t i = gtid; i < y_vec4; i += nthreads) y_zero[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0 && bslot < 1024) TC_STAMP(ts, bslot, 2);
}

// Ragged feature counts: K6 wrote Y padded to rx columns; copy the first rows_x of each row.
__global__ void __launch_bounds__(256) stream_tc_unpad_kernel(const int32_t* __restrict__ src,
                                                              int32_t* __restrict__ dst, uint32_t rx,
                                                              uint32_t rows_x, uint64_t n) {
  pdl_trigger();
  pdl_wait();
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / rows_x;
    dst[i] = src[r * rx + (i - r * rows_x)];
  }
}

struct Layout {
  uint32_t n_mma, wst, bst, w_off, st_off, smem;
  bool pw;  // pair-box weight layout
};
// The pair-box layout (two step boxes in flight per row group) where shared memory allows it,
// else one 16-row box per warp.
Layout layout_of(uint64_t rows_x, int n_w, uint32_t wst_cap = kMaxWst, bool allow_pw = true) {
  Layout l{};
  l.n_mma = n_mma_of(static_cast<uint32_t>(rows_x));
  for (int pw = allow_pw ? 1 : 0; pw >= 0; --pw) {
    l.pw = pw != 0;
    for (uint32_t bst = kBStages; bst >= 2; --bst) {
      l.bst = bst;
      l.w_off = bst * b_stage_bytes(l.n_mma);
      for (uint32_t wst = pw ? 1u : wst_cap; wst >= 1; --wst) {
        l.wst = wst;
        l.st_off = l.w_off + (pw ? 8u * kPairSlots * pslot_bytes(n_w) : kTfWarps * wst * wslot_bytes(n_w));
        l.smem = l.st_off + kEpiWarps * kStageBytes + 1024u;  // + alignment slack
        if (l.smem <= kSmemCap) return l;
      }
    }
  }
  l.smem = 0;
  return l;
}
// feature code words: whole steps, whole step pairs for the pair layout
uint32_t kwords_of(uint64_t k, bool pw = true) {
  const uint64_t unit = (pw ? 2u : 1u) * kStepBytes;
  return static_cast<uint32_t>((k + unit - 1) / unit * (unit / 32u));
}
uint32_t prep_blocks_of(uint64_t k) { return (kwords_of(k) + kPrepThreads - 1) / kPrepThreads; }

template <int N, bool PW>
cudaError_t launch_n(const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap& ty, const TcParams& p,
                     unsigned grid, uint32_t smem, cudaStream_t s) {
  auto kern = stream_tc_kernel<N, PW>;
  static DeviceBits attr_set;
  const int dev = current_device();
  if (!attr_set.test(dev)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemCap));
    if (e != cudaSuccess) return e;
    attr_set.set(dev);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tw, tx, ty, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

bool stream_tc_supported(const uint32_t* w, uint64_t rows_w, uint64_t rows_x, uint64_t k, int n_w,
                         const void* y) {
  const uint64_t wpr = (k + 31) / 32;
  const uint64_t tiles = (rows_w + kTileRows - 1) / kTileRows;
  const uint64_t steps = (wpr + kStepWords - 1) / kStepWords;
  const uint64_t rx4 = (rows_x + 3) / 4 * 4;
  return rows_x >= 1 && rx4 <= kMaxRowsX && n_w <= 4 && wpr % 4 == 0 &&
         reinterpret_cast<uintptr_t>(w) % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 4 == 0 &&
         tiles * steps < 65536 && layout_of(rx4, n_w).smem != 0;
}

bool stream_tc_padded(uint64_t rows_x, const void* y) {
  return rows_x % 4 != 0 || reinterpret_cast<uintptr_t>(y) % 16 != 0;
}

size_t stream_tc_ws_bytes(uint64_t rows_x, uint64_t k, uint64_t rows_w, bool padded) {
  const uint64_t rx4 = (rows_x + 3) / 4 * 4;
  const uint64_t n_mma = n_mma_of(static_cast<uint32_t>(rx4));
  return round_up(n_mma * kwords_of(k) * 32u, 256) + round_up(n_mma * prep_blocks_of(k) * 4u, 256) +
         (padded ? round_up(rows_w * rx4 * 4u, 256) : 0);
}

cudaError_t launch_stream_tc(const StreamTcArgs& a, cudaStream_t s) {
  static const uint32_t wst_cap = [] {  // dev A/B: APMM_TC_WST caps the weight ring depth
    const char* e = APMM_DEV_ENV("APMM_TC_WST");
    return e ? static_cast<uint32_t>(std::atoi(e)) : kMaxWst;
  }();
  static const bool allow_pw = APMM_DEV_ENV("APMM_TC_NOPAIR") == nullptr;  // dev A/B
  // ragged feature counts run on a 4-aligned row count into a padded Y in the workspace
  const bool padded = stream_tc_padded(a.rows_x, a.y);
  const uint64_t rx = (a.rows_x + 3) / 4 * 4;
  Layout l = layout_of(rx, a.n_w, wst_cap, allow_pw);
  if (!l.smem) return cudaErrorInvalidConfiguration;
  const uint32_t wpr = static_cast<uint32_t>((a.k + 31) / 32);
  if (l.pw) {
    // stream-K over step pairs is coarser: keep the pair layout only where it does not lengthen
    // the busiest CTA's step count (11008 x 16 x 4096: 6 steps vs 5 measured 12% slower)
    const uint64_t tl = (a.rows_w + kTileRows - 1) / kTileRows, sms = static_cast<uint64_t>(a.num_sms);
    const uint64_t n1 = tl * (kwords_of(a.k, false) / kStepWords), n2 = tl * (kwords_of(a.k, true) / kStepWords) / 2;
    const uint64_t max1 = (n1 + sms - 1) / sms, max2 = 2 * ((n2 + sms - 1) / sms);
    if (max2 > max1) l = layout_of(rx, a.n_w, wst_cap, false);
  }
  const uint32_t kwords = kwords_of(a.k, l.pw);
  const uint32_t spt = kwords / kStepWords;
  const uint32_t tiles = static_cast<uint32_t>((a.rows_w + kTileRows - 1) / kTileRows);
  const uint32_t total = tiles * spt / (l.pw ? 2u : 1u);  // work units: steps or step pairs
  const uint32_t grid = total < static_cast<uint32_t>(a.num_sms) ? total : static_cast<uint32_t>(a.num_sms);
  uint8_t* codes = static_cast<uint8_t*>(a.ws);
  int32_t* rsx_part = reinterpret_cast<int32_t*>(codes + round_up(uint64_t(l.n_mma) * kwords * 32u, 256));
  const uint32_t parts = prep_blocks_of(a.k);
  int32_t* ydst = padded ? reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(rsx_part) +
                                                       round_up(uint64_t(l.n_mma) * parts * 4u, 256))
                         : a.y;

  // feature prep (+ Y zeroing)
  {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(parts, l.n_mma);
    cfg.blockDim = dim3(kPrepThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const uint64_t y_vec4 = a.rows_w * rx / 4;
    cudaError_t e = cudaLaunchKernelEx(&cfg, stream_tc_prep_kernel, a.x_planes,
                                       static_cast<uint32_t>(rx), static_cast<uint32_t>(a.rows_x), wpr,
                                       a.n_x, kwords, codes, rsx_part, reinterpret_cast<uint4*>(ydst), y_vec4,
                                       a.early_x ? 1u : 0u, a.trace_prep);
    if (e != cudaSuccess) return e;
  }
  CUtensorMap tw, tx, ty;
  {
    const uint64_t dims[3] = {wpr, a.rows_w, static_cast<uint64_t>(a.n_w)};
    const uint64_t strides[2] = {uint64_t(wpr) * 4, uint64_t(wpr) * 4 * a.rows_w};
    const uint32_t box[3] = {(l.pw ? 2u : 1u) * kStepWords, kItemRows, static_cast<uint32_t>(a.n_w)};
    if (encode_tmap_3d_u32(&tw, a.w_planes, dims, strides, box) != CUDA_SUCCESS) {
      return cudaErrorInvalidValue;
    }
  }
  if (encode_tmap_2d(&tx, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, codes, uint64_t(kwords) * 32u, l.n_mma,
                     uint64_t(kwords) * 32u, 128u, l.n_mma) != CUDA_SUCCESS) {
    return cudaErrorInvalidValue;
  }
  if (encode_tmap_2d(&ty, CU_TENSOR_MAP_DATA_TYPE_INT32, 4, ydst, rx, a.rows_w, rx * 4,
                     32u, 32u) != CUDA_SUCCESS) {
    return cudaErrorInvalidValue;
  }
  TcParams p{};
  p.rsx_part = rsx_part;
  p.parts = parts;
  p.rows_x = static_cast<uint32_t>(rx);
  p.n_mma = l.n_mma;
  p.n_w = static_cast<uint32_t>(a.n_w);
  p.steps_per_tile = spt;
  p.q_steps = total / grid;
  p.r_steps = total % grid;
  p.inv_spt = ((uint64_t(1) << 32) + spt - 1) / spt;
  p.wst = l.wst;
  p.bst = l.bst;
  p.w_off = l.w_off;
  p.st_off = l.st_off;
  const uint32_t A = (1u << a.n_w) - 1u, B = (1u << a.n_x) - 1u;
  p.coef_w = 2u * B;
  p.coef_x = 2u * A;
  p.c0 = static_cast<uint32_t>(a.k) * A * B;
  p.early_w = a.early_w ? 1u : 0u;
  p.ts = a.trace;
  // two D accumulators where tensor memory holds them (A buffers at 0..255): the epilogue of a
  // segment then overlaps the next segment's MMAs
  static const bool nd1 = APMM_DEV_ENV("APMM_TC_ND1") != nullptr;  // dev A/B
  p.dstride = (l.n_mma + 31u) / 32u * 32u;
  const uint32_t dread = ((static_cast<uint32_t>(rx) + 31u) / 32u) * 32u;
  p.nd = !nd1 && kColD + p.dstride + (dread > l.n_mma ? dread : l.n_mma) <= kTmemCols ? 2u : 1u;
  static const uint32_t ts_mode = [] {
    const char* e = APMM_DEV_ENV("APMM_TC_TS_MODE");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
  }();
  p.ts_mode = ts_mode;
  static const uint32_t ablate = [] {
    const char* e = APMM_DEV_ENV("APMM_TC_ABLATE");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
  }();
  p.ablate = ablate;
  if (a.ev_start) cudaEventRecordWithFlags(a.ev_start, s, a.ev_flags);
  cudaError_t e;
  switch (a.n_w) {
    case 1: e = l.pw ? launch_n<1, true>(tw, tx, ty, p, grid, l.smem, s) : launch_n<1, false>(tw, tx, ty, p, grid, l.smem, s); break;
    case 2: e = l.pw ? launch_n<2, true>(tw, tx, ty, p, grid, l.smem, s) : launch_n<2, false>(tw, tx, ty, p, grid, l.smem, s); break;
    case 3: e = l.pw ? launch_n<3, true>(tw, tx, ty, p, grid, l.smem, s) : launch_n<3, false>(tw, tx, ty, p, grid, l.smem, s); break;
    default: e = l.pw ? launch_n<4, true>(tw, tx, ty, p, grid, l.smem, s) : launch_n<4, false>(tw, tx, ty, p, grid, l.smem, s); break;
  }
  if (e == cudaSuccess && padded) {
    // padded Y -> the caller's [rows_w][rows_x] (PDL: waits for K6 inside)
    cudaLaunchConfig_t cfg{};
    const uint64_t n = a.rows_w * a.rows_x;
    cfg.gridDim = dim3(static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4u * a.num_sms)));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, stream_tc_unpad_kernel, static_cast<const int32_t*>(ydst), a.y,
                           static_cast<uint32_t>(rx), static_cast<uint32_t>(a.rows_x), n);
  }
  if (a.ev_stop) cudaEventRecordWithFlags(a.ev_stop, s, a.ev_flags);
  return e;
}

}  // namespace apmm_b200
