// skinny.cu -- K5: the WnAm bipolar-INT GEMM for few feature rows (decode / small-M LLM
// shapes), HBM-bound on the packed weight planes. Two launches per matmul_ap call: a tiny
// feature-prep kernel (X planes -> MMA fragment order, once) and the streaming kernel; for a
// single feature row the streaming kernel builds its X slice itself (one launch).
//
// Why a separate path. With M_tok < 64 the GEMM does ~2*M ops per weight code, so the
// roofline is the HBM read of the packed weight planes (n_w bits per weight). The large-M
// path (expand -> u8 codes in HBM -> tcgen05 GEMM) would write and re-read 8/n_w times
// those bytes. Here every warp streams its weight tiles (16 rows x 512 columns x n_w
// planes) from HBM with its own TMA ring in shared memory, turns them into u8 code
// fragments in registers by a partial 8x8 bit transpose, and feeds legacy-pipe mma.sync
// m16n8k32 u8 x u8 -> s32 MMAs (measured ~1.1 POPS on this part, scripts/imma_probe.cu:
// far above what M < 64 needs). What bounds it besides HBM is the instruction count per
// weight code: the transpose costs ~0.7 ops/code for n_w <= 4 (~0.4 for n_w <= 2, see EXT)
// and is split over the ALU and FMA pipes (shifts as IMAD / IMAD.HI), rowsum(U_w) comes out
// of the MMA through an all-ones feature column (no POPC), and the loop has no divisions.
//
// The algebra is the same as the large-M path: one u8 x u8 MMA
// of the unsigned codes performs the whole 2^(i+j)-weighted plane-pair recovery of the
// reference's matmul_ap (kernel.cpp:187-254); the rank-1 term is applied in the epilogue:
//   Y = 4 * sum_k u_w u_x - 2B * rowsum(U_w) - 2A * rowsum(U_x) + K*A*B   (mod 2^32).
// The first two terms are linear in K, so each K slice contributes 4*S_s - 2B*rsw_s; the
// slice-0 CTAs add the X term and the constant once.
//
// Fragment mapping (PTX m16n8k32 .u8): thread (g = lane/4, t = lane%4) supplies A rows g
// and g+8 and B column g at K slots {4t+b, 16+4t+b}. The K order inside the MMA is free as
// long as A and B agree, and the slot -> column map below depends only on (t, slot), never
// on g:
//   thread t takes plane words [16c + 4t, +4) (128 columns) of its two weight rows;
//   a 32-column word is bit-transposed so that register r, byte B holds column 8B + r;
//   the prep kernel transposes X the same way, so the B fragment of the MMA that uses A
//   registers (r, r+1) is X's registers (r, r+1) of the same word.
// For n_w <= 4 only two of the three delta-swap stages run on W: register r (r < 4) then
// holds column 8B+r in its low nibble and column 8B+4+r in its high nibble.
// `x & 0x0F0F0F0F` gives the first, `x - lo` gives 16x the second; the latter goes into a
// separate accumulator that is divided by 16 at the end (exact: the host admits this
// variant only when K*(2^n_w-1)*(2^n_x-1) < 2^28, so 16x any partial sum fits in 32 bits).
//
// Work split (host planner, plan_for): K is cut into S slices of whole 512-column chunks;
// a persistent CTA owns one slice for its lifetime (one bulk copy stages its X slice in
// shared memory) and walks a strided list of row tiles of 16*R weight rows. Its warps are
// R row groups x (warps/R) K groups; the K groups' partial sums meet in shared memory
// (red.shared.add). With S == 1 the CTA applies the recovery / dequant epilogue and
// writes Y directly. With S > 1 partial sums go to an int32 workspace with wrapping
// atomics (exact mod 2^32, order-independent); the last CTA of a tile (counter)
// finalises it and re-zeroes the workspace for the next call.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "ptx.cuh"

namespace apmm_b200 {
namespace {

constexpr int kChunkWords = 16;  // 512 columns per warp step
constexpr uint32_t kSkSmemSM = 224u * 1024u;  // dynamic budget per SM (227 KB max minus static)
constexpr int kPrepThreads = 256;
constexpr uint64_t kInprepMaxRows = 8;  // feature rows staged by the streaming kernel itself

// One persistent CTA per SM: 16 warps where registers allow, else 8. (Two smaller CTAs per
// SM were measured slower: the halved shared memory forces more K slices, and the split-K
// finalisation tail costs more than the earlier start of the next call gains.)
__host__ __device__ constexpr int sk_threads(int n, int nt) { return (n <= 3 && nt <= 4) ? 512 : 256; }
__host__ __device__ constexpr int sk_ctas_per_sm(int, int) { return 1; }
__host__ __device__ constexpr uint32_t sk_smem_budget(int n, int nt) {
  return kSkSmemSM / sk_ctas_per_sm(n, nt);
}
// Per-warp TMA ring: a slot holds one work item, n planes x 16 rows x 64 B = n KB. Two slots
// per warp: with deeper rings every warp requests its whole share at once, HBM serves the
// requests in arbitrary order and warps wait for their first item while later items arrive
// (8192^2 W3A8 M=1: 9.4 us at depth 2, 10.1 at 3, 10.8 at 4 or 8,
// profiles/r02/r2_sk_stages.txt, profiles/r02/r2_decode_xfirst.txt); 16 warps x 2 slots keep
// ~100 KB per SM in flight.
#ifndef APMM_SK_STAGES_DEV
constexpr uint32_t kStages = 2;
#else
constexpr uint32_t kStages = APMM_SK_STAGES_DEV;  // dev A/B builds only
#endif
constexpr int kXPieces = 16;  // X slice copy pieces (barriers)
__host__ __device__ constexpr uint32_t slot_bytes(int n) { return static_cast<uint32_t>(n) * 1024u; }
// Shared-memory X layout per 512-column chunk, real feature rows only (M = rows_x):
// [w 0..3][half 0..1][feature row 0..M-1][t 0..3] x 16 B. Thread (g, t) of n-tile nt
// takes feature row nt*8+g, word 16*chunk + 4t + w, code registers [4h, 4h+4) (register
// r, byte B = code of column 8B + r). A warp's 128-bit reads are 512 contiguous bytes.
// Rows >= M are zero codes and the all-ones column (slot 8*NT-1) is a register constant.
__host__ __device__ constexpr uint32_t chunk_bytes_m(uint32_t m) { return 512u * m; }
// Fragment rows per chunk: the real feature rows, then a zero row and an all-ones row, so
// that every lane's B fragment is a plain shared load (lanes of padded MMA columns point at
// the zero row, the rowsum column at the ones row; no per-MMA register moves).
__host__ __device__ constexpr uint32_t frag_rows(uint32_t rows_x) { return rows_x + 2u; }
// cross-warp reduction buffer: [16 R][m_pad] u32, R <= 8
__host__ __device__ constexpr uint32_t red_bytes(int nt, uint32_t r) { return 16u * r * nt * 8u * 4u; }

struct SkinnyParams {
  const uint8_t* xfrag;      // prep output: [chunks_total][chunk_bytes_m(frag_rows(rows_x))]
  const uint32_t* x_planes;  // inprep: reference layout [n_x][rows_x][wpr]
  uint32_t inprep;           // 1: this kernel builds its X slice itself (no prep kernel)
  uint32_t n_x, k_logical;
  // work split, precomputed on the host so that the prologue has no division: a CTA's first
  // TMA issue is on the critical path of every call
  uint32_t log2_wk;          // warps_k = WARPS >> log2(R), a power of two
  uint32_t gs, cpw, xpc;     // CTAs per slice, chunks per warp per tile, chunks per X piece
  uint64_t inv_slices, inv_gs, inv_xpc;  // ceil(2^32 / d) for d = S, gs, xpc
  uint64_t inv_sw, inv_sw_last;  // the same for the slice words (full slices, the last slice)
  const int32_t* rsx;        // prep output: rowsum(U_x) parts [rows_x][rsx_parts]
  uint32_t rsx_parts;
  uint32_t rows_w, rows_x, wpr, n_planes;
  uint32_t chunks_total;     // ceil(wpr / 16)
  uint32_t slices, slice_chunks;
  uint32_t rgroups;          // R: 16-row groups per tile (warps_k = warps / R)
  uint32_t n_tiles;          // ceil(rows_w / (16 R))
  uint32_t ring_off, red_off;  // shared-memory carve-up (bytes)
  uint32_t* acc;             // S > 1: [n_tiles * 16R][m_pad], zero on entry and exit
  uint32_t* counters;        // S > 1: [n_tiles]
  int32_t* y;
  float* yf;
  const double* s_w;
  const double* s_x;
  int gran_w, gran_x;
  uint32_t coef_w, coef_x, c0;
  // multipliers kept in the parameter bank so ptxas emits IMAD (FMA pipe), not SHF/IADD
  uint32_t m2, m4, m16, neg1;
  unsigned long long* ts;    // dev builds only: per-CTA phase stamps [grid][8], else null
  uint32_t early_w;          // PDL: weight loads may start before the previous kernel completes
  uint32_t ts_clock;         // dev: stamps are the SM's clock64 (cycles, per CTA), else globaltimer
  uint32_t x_first;          // dev A/B (APMM_SK_XFIRST): in-kernel prep issues its feature loads
                             // before the first weight load (which then waits for pdl_wait)
};

// floor(n / d) for n, d < 2^16 from inv = ceil(2^32 / d): exact (the error n * (inv * d - 2^32)
// / 2^32 stays below 1 / d)
APMM_DEV uint32_t div_small(uint32_t n, uint64_t inv) {
  return static_cast<uint32_t>((static_cast<uint64_t>(n) * inv) >> 32);
}
inline uint64_t inv_small(uint32_t d) { return ((uint64_t(1) << 32) + d - 1) / d; }

// dev builds: per-CTA phase stamps (0 start, 1 pdl_wait, 2 x_ready, 3 item0, 4 tile0, 5 end,
// 6 inited, 7 issued); compiled out of the release library
#ifdef APMM_DEVTOOLS
#define SK_STAMP(k)                                                                         \
  do {                                                                                      \
    if (p.ts && tid == 0)                                                                   \
      p.ts[blockIdx.x * 8 + (k)] =                                                          \
          p.ts_clock ? static_cast<unsigned long long>(clock64()) : gtime_ns();             \
  } while (0)
#else
#define SK_STAMP(k) \
  do {              \
  } while (0)
#endif

#ifdef APMM_DEVTOOLS
APMM_DEV unsigned long long gtime_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

APMM_DEV void mma_u8(uint32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                     uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

APMM_DEV void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar, int32_t c0, int32_t c1,
                          int32_t c2, uint64_t hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "l"(hint)
      : "memory");
}
// One bulk (non-tensor) TMA copy global -> this CTA's shared memory, completing on `bar`.
APMM_DEV void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
APMM_DEV uint32_t mulhi(uint32_t a, uint32_t b) { return __umulhi(a, b); }

// Delta swap in select form with both shifts on the FMA pipe (IMAD / IMAD.HI) and the two
// selects as LOP3 on the ALU pipe.
// sel(a, b, m) = (a & ~m) | (b & m) as one LOP3 (written in PTX so the compiler keeps the
// select form instead of re-associating it into AND/OR chains around the multiplies).
template <uint32_t M>
APMM_DEV uint32_t sel(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(r) : "r"(a), "r"(b), "n"(M));
  return r;
}
template <int S>
APMM_DEV void swap_sel(uint32_t& a, uint32_t& b, uint32_t m, uint32_t mul_s) {
  const uint32_t bs = b * mul_s;                      // b << S
  const uint32_t as = mulhi(a, 1u << (32 - S));       // a >> S
  const uint32_t na = S == 1 ? sel<0xAAAAAAAAu>(a, bs) : S == 2 ? sel<0xCCCCCCCCu>(a, bs)
                                                                : sel<0xF0F0F0F0u>(a, bs);
  b = S == 1 ? sel<0x55555555u>(b, as) : S == 2 ? sel<0x33333333u>(b, as) : sel<0x0F0F0F0Fu>(b, as);
  a = na;
  (void)m;
}

// Codes of one 32-column word (x[i] = plane i word, zero for i >= N). SPLIT (N <= 4):
// o[r] = codes of columns 8B+r, o[4+r] = 16x codes of columns 8B+4+r (r < 4). Otherwise
// o[r] = codes of columns 8B+r (r < 8).
// EXT (N <= 2, few n-tiles): a single distance-1 swap leaves 2-bit codes; o[2s], o[2s+1]
// = 4^s x codes of columns 8B+2s, 8B+2s+1 (s < 4), summed into four scaled accumulators --
// 12 ops per word instead of ~22 for the nibble split.
template <int N, bool SPLIT, bool EXT = false>
APMM_DEV void codes_of_word(uint32_t (&x)[8], uint32_t (&o)[8], const SkinnyParams& p) {
  if (EXT) {
    swap_sel<1>(x[0], x[1], 0x55555555u, p.m2);  // x[0]: cols 8B+{0,2,4,6}, x[1]: 8B+{1,3,5,7}
    o[0] = x[0] & 0x03030303u;
    o[1] = x[1] & 0x03030303u;
    o[2] = x[0] & 0x0C0C0C0Cu;
    o[3] = x[1] & 0x0C0C0C0Cu;
    o[4] = x[0] & 0x30303030u;
    o[5] = x[1] & 0x30303030u;
    o[6] = x[0] & 0xC0C0C0C0u;
    o[7] = x[1] & 0xC0C0C0C0u;
  } else if (SPLIT) {
    swap_sel<2>(x[0], x[2], 0x33333333u, p.m4);
    swap_sel<2>(x[1], x[3], 0x33333333u, p.m4);
    swap_sel<1>(x[0], x[1], 0x55555555u, p.m2);
    swap_sel<1>(x[2], x[3], 0x55555555u, p.m2);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      o[r] = x[r] & 0x0F0F0F0Fu;
      o[4 + r] = o[r] * p.neg1 + x[r];  // x - lo = the high nibbles, 16x
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) swap_sel<4>(x[i], x[i + 4], 0x0F0F0F0Fu, p.m16);
#pragma unroll
    for (int i = 0; i < 8; i += 4) {
      swap_sel<2>(x[i], x[i + 2], 0x33333333u, p.m4);
      swap_sel<2>(x[i + 1], x[i + 3], 0x33333333u, p.m4);
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2) swap_sel<1>(x[i], x[i + 1], 0x55555555u, p.m2);
#pragma unroll
    for (int r = 0; r < 8; ++r) o[r] = x[r];
  }
}

// Plain 8x8 transpose for the prep kernel (register r, byte B <- column 8B + r).
APMM_DEV void transpose8(uint32_t (&x)[8]) {
  auto sw = [](uint32_t& a, uint32_t& b, int s, uint32_t m) {
    const uint32_t na = (a & ~(m << s)) | ((b << s) & (m << s));
    b = (b & ~m) | ((a >> s) & m);
    a = na;
  };
#pragma unroll
  for (int i = 0; i < 4; ++i) sw(x[i], x[i + 4], 4, 0x0F0F0F0Fu);
#pragma unroll
  for (int i = 0; i < 8; i += 4) {
    sw(x[i], x[i + 2], 2, 0x33333333u);
    sw(x[i + 1], x[i + 3], 2, 0x33333333u);
  }
#pragma unroll
  for (int i = 0; i < 8; i += 2) sw(x[i], x[i + 1], 1, 0x55555555u);
}

// ---- feature prep: X planes -> fragment-order codes + rowsum(U_x) -----------------------
// grid (ceil(chunks_total*16 / 256), rows_x); thread = (feature row, 32-column word).
// PDL: triggers its dependents at once (the streaming kernel's weight loads may start). It
// reads the caller's X planes only after griddepcontrol.wait (X may be the output of the
// previous kernel in the stream) unless early_x (APMM_OPT_EARLY_FEATURE_READ), and writes
// its workspace half only after it.
__global__ void __launch_bounds__(kPrepThreads) prep_x_kernel(const uint32_t* __restrict__ x,
                                                              uint32_t rows_x, uint32_t wpr,
                                                              int n_x, uint32_t words_pad,
                                                              uint8_t* __restrict__ xfrag,
                                                              int32_t* __restrict__ rsx_part,
                                                              uint32_t early_x) {
  apmm_ptx::pdl_trigger();
  if (!early_x) apmm_ptx::pdl_wait();
  const uint32_t tok = blockIdx.y, W = blockIdx.x * kPrepThreads + threadIdx.x;
  const uint32_t xr = frag_rows(rows_x);
  uint32_t v[8];
  int32_t rs = 0;
  const uint64_t pstride = uint64_t(rows_x) * wpr;
  const bool real = tok < rows_x;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = (real && i < n_x && W < wpr) ? __ldg(x + i * pstride + uint64_t(tok) * wpr + W)
                                        : (tok == rows_x + 1u ? 0x01010101u : 0u);
    if (real && i < n_x) rs += __popc(v[i]) << i;
  }
  if (real) transpose8(v);
  if (early_x) apmm_ptx::pdl_wait();  // the workspace half may be written only now
  if (W < words_pad) {
    const uint32_t cl = W / kChunkWords, t = (W % kChunkWords) >> 2, w = W & 3u;
    uint4* dst = reinterpret_cast<uint4*>(xfrag + uint64_t(cl) * chunk_bytes_m(xr)) +
                 ((w * 2u) * xr + tok) * 4u + t;
    dst[0] = make_uint4(v[0], v[1], v[2], v[3]);
    dst[xr * 4u] = make_uint4(v[4], v[5], v[6], v[7]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
  __shared__ int32_t part[kPrepThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = rs;
  __syncthreads();
  if (threadIdx.x == 0 && real) {
    int32_t s = 0;
    for (int i = 0; i < kPrepThreads / 32; ++i) s += part[i];
    rsx_part[uint64_t(tok) * gridDim.x + blockIdx.x] = s;
  }
}

// PR: rowsum(U_w) from popcounts of the weight planes instead of an all-ones feature column
// (used when the feature rows fill their n-tiles exactly: M_tok = 8 needs one n-tile, not two)
template <int N, int NT, bool SPLIT, bool PR>
__global__ void __launch_bounds__(sk_threads(N, NT), sk_ctas_per_sm(N, NT))
    skinny_kernel(const __grid_constant__ CUtensorMap tmap_w, const SkinnyParams p) {
  constexpr int THREADS = sk_threads(N, NT);
  constexpr int WARPS = THREADS / 32;
  constexpr uint32_t SLOT = slot_bytes(N);
  constexpr uint32_t M_PAD = NT * 8u;
  constexpr uint32_t ONES = PR ? 0xFFFFFFFFu : M_PAD - 1u;  // the all-ones column -> rowsum(U_w)
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[WARPS * kStages];
  __shared__ __align__(8) uint64_t xbars[kXPieces];  // X slice arrival, per piece of chunks
  __shared__ uint32_t rsx_s[M_PAD];
  __shared__ uint32_t rsw_s[PR ? 128 : 1];  // PR: rowsum(U_w) of the tile's rows
  __shared__ uint32_t s_last;

  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t g = lane >> 2, t = lane & 3;
  SK_STAMP(0);
  if (tid == 0) apmm_ptx::tma_prefetch_desc(&tmap_w);  // the descriptor fetch off every warp's first load
  const uint32_t warps_k = 1u << p.log2_wk;
  const uint32_t wr = warp >> p.log2_wk, wk = warp & (warps_k - 1u);
  const uint32_t tile_rows = (WARPS >> p.log2_wk) * 16u;

  // persistent CTA: slice = blockIdx.x % S, tiles j0, j0 + gs, ... (gs CTAs per slice)
  const uint32_t j0 = div_small(blockIdx.x, p.inv_slices);
  const uint32_t slice = blockIdx.x - j0 * p.slices;
  const uint32_t gs = p.gs, cpw = p.cpw;  // chunks per warp per tile
  const uint32_t s_begin = slice * p.slice_chunks;
  const uint32_t s_end = min(s_begin + p.slice_chunks, p.chunks_total);
  const uint32_t my_tiles = j0 < p.n_tiles ? div_small(p.n_tiles - j0 + gs - 1u, p.inv_gs) : 0u;

  uint8_t* xs = smem;
  const uint32_t ring = apmm_ptx::smem_u32(smem + p.ring_off) + warp * (kStages * SLOT);
  uint32_t* red = reinterpret_cast<uint32_t*>(smem + p.red_off);  // [tile_rows][M_PAD]
  uint64_t* bars = full_bar + warp * kStages;
  const uint32_t xchunk_bytes = chunk_bytes_m(frag_rows(p.rows_x));

  // ---- per-warp TMA ring: item cursor (tile index, chunk step) ----
  uint32_t is_tile = 0, is_c = 0, is_slot = 0;
  uint64_t hint = 0;
  auto issue = [&]() {
    if (is_tile < my_tiles) {
      const uint32_t chunk = s_begin + is_c * warps_k + wk;
      if (chunk < s_end && lane == 0) {
        const uint32_t row0 = (j0 + is_tile * gs) * tile_rows + wr * 16u;
        apmm_ptx::mbar_arrive_expect_tx(&bars[is_slot], p.n_planes * 1024u);
        tma_load_3d(ring + is_slot * SLOT, &tmap_w, apmm_ptx::smem_u32(&bars[is_slot]),
                    int32_t(chunk * kChunkWords), int32_t(row0), 0, hint);
      }
      if (++is_c == cpw) { is_c = 0; ++is_tile; }
    }
    is_slot = is_slot + 1u == kStages ? 0u : is_slot + 1u;
  };

  // Each warp initialises its own ring barriers and issues its first weight load at once:
  // the weight planes are inputs of this call, so their loads may overlap the kernel still
  // running ahead of us (PDL); X, the workspace and Y only after pdl_wait.
  if (lane == 0) {
#pragma unroll
    for (uint32_t q = 0; q < kStages; ++q) apmm_ptx::mbar_init(&bars[q], 1);
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < kXPieces; ++i) apmm_ptx::mbar_init(&xbars[i], 1);
    }
    // mbarrier inits -> visible to the TMA unit (async proxy). A non-cluster launch needs
    // no cluster-scope release (fence.mbarrier_init.release.cluster cost ~0.8 us per CTA at
    // kernel start, profiles/r01b_skinny_phase_ts2.txt).
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  SK_STAMP(6);
  hint = apmm_ptx::policy_evict_first();  // weights are read exactly once
  if (!p.early_w) apmm_ptx::pdl_wait();  // weights may be produced by the previous kernel
  const bool x_first = p.x_first && p.inprep;
  if (!x_first)
#pragma unroll
    for (uint32_t q = 0; q + 1 < kStages; ++q) issue();
  SK_STAMP(7);
  apmm_ptx::pdl_wait();
  SK_STAMP(1);
  __syncthreads();  // xbars initialised
  const uint32_t xpc = p.xpc;  // chunks per X piece
  if (p.inprep) {
    // Feature prep in the prologue (few feature rows): this CTA's K slice of X planes ->
    // fragment-order codes in shared memory, its rowsum(U_x) share, and the zero / ones
    // rows. One thread per (feature row, 32-column word): n_x words -> 8x8 transpose. Every
    // thread's first loads are issued before anything else, so the whole slice of a single
    // feature row costs one round trip; the constant rows need no loads.
    const uint32_t slice_words = (s_end > s_begin ? s_end - s_begin : 0u) * kChunkWords;
    const uint32_t xr = frag_rows(p.rows_x);
    const uint32_t real_words = p.rows_x * slice_words;
    const uint64_t pstride = uint64_t(p.rows_x) * p.wpr;
    const uint64_t inv_sw = slice + 1u == p.slices ? p.inv_sw_last : p.inv_sw;
    auto xload = [&](uint32_t idx, uint32_t (&v)[8]) {
      const uint32_t tok = div_small(idx, inv_sw), wl = idx - tok * slice_words;
      const uint32_t W = s_begin * kChunkWords + wl;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[i] = (uint32_t(i) < p.n_x && W < p.wpr)
                   ? __ldg(p.x_planes + i * pstride + uint64_t(tok) * p.wpr + W) : 0u;
    };
    auto xstore = [&](uint32_t tok, uint32_t wl, const uint32_t (&v)[8]) {
      const uint32_t cl = wl / kChunkWords, t4 = (wl % kChunkWords) >> 2, w = wl & 3u;
      uint4* dst = reinterpret_cast<uint4*>(xs + cl * xchunk_bytes) + ((w * 2u) * xr + tok) * 4u + t4;
      dst[0] = make_uint4(v[0], v[1], v[2], v[3]);
      dst[xr * 4u] = make_uint4(v[4], v[5], v[6], v[7]);
    };
    auto xprocess = [&](uint32_t idx, uint32_t (&v)[8]) {
      const uint32_t tok = div_small(idx, inv_sw), wl = idx - tok * slice_words;
      uint32_t rs = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) rs += uint32_t(__popc(v[i])) << i;
      transpose8(v);
      xstore(tok, wl, v);
      if (rs) atomicAdd(&rsx_s[tok], rs);
    };
    uint32_t v0[8], v1[8];
    if (tid < real_words) xload(tid, v0);
    if (tid + THREADS < real_words) xload(tid + THREADS, v1);
    if (x_first)
#pragma unroll
      for (uint32_t q = 0; q + 1 < kStages; ++q) issue();
    for (uint32_t q = tid; q < M_PAD; q += THREADS) rsx_s[q] = 0u;
    for (uint32_t q = tid; q < tile_rows * M_PAD; q += THREADS) red[q] = 0u;
    if (PR) for (uint32_t q = tid; q < tile_rows; q += THREADS) rsw_s[q] = 0u;
    for (uint32_t q = tid; q < 2u * slice_words; q += THREADS) {  // the zero and all-ones rows
      const uint32_t hi = q >= slice_words ? 1u : 0u, c = hi ? 0x01010101u : 0u;
      const uint32_t v[8] = {c, c, c, c, c, c, c, c};
      xstore(p.rows_x + hi, q - hi * slice_words, v);
    }
    __syncthreads();  // rsx_s zeroed
    if (tid < real_words) xprocess(tid, v0);
    if (tid + THREADS < real_words) xprocess(tid + THREADS, v1);
    for (uint32_t idx = tid + 2 * THREADS; idx < real_words; idx += 2 * THREADS) {
      uint32_t v[8], v2[8];
      const bool two = idx + THREADS < real_words;
      xload(idx, v);
      if (two) xload(idx + THREADS, v2);
      xprocess(idx, v);
      if (two) xprocess(idx + THREADS, v2);
    }
    __syncthreads();
  } else {
    const uint32_t xbytes = (s_end > s_begin ? s_end - s_begin : 0u) * xchunk_bytes;
    if (tid == 0) {
      // one bulk copy (and barrier) per piece of `xpc` chunks, so warps start on their
      // first chunk while the rest of the slice is still arriving
      const uint8_t* src = p.xfrag + uint64_t(s_begin) * xchunk_bytes;
      const uint32_t piece = xpc * xchunk_bytes;
      for (uint32_t off = 0, i = 0; off < xbytes; off += piece, ++i) {
        const uint32_t b = min(piece, xbytes - off);
        apmm_ptx::mbar_arrive_expect_tx(&xbars[i], b);
        for (uint32_t o2 = 0; o2 < b; o2 += 32768u) {
          bulk_g2s(apmm_ptx::smem_u32(xs + off + o2), src + off + o2, min(32768u, b - o2),
                   apmm_ptx::smem_u32(&xbars[i]));
        }
      }
    }
    // slice 0 adds the X term of the whole K (prep kernel's rowsum parts)
    for (uint32_t q = tid; q < M_PAD; q += THREADS) {
      int32_t s = 0;
      if (slice == 0 && q < p.rows_x) {
        for (uint32_t k = 0; k < p.rsx_parts; ++k) s += __ldg(p.rsx + uint64_t(q) * p.rsx_parts + k);
      }
      rsx_s[q] = static_cast<uint32_t>(s);
    }
    for (uint32_t q = tid; q < tile_rows * M_PAD; q += THREADS) red[q] = 0u;
    if (PR) for (uint32_t q = tid; q < tile_rows; q += THREADS) rsw_s[q] = 0u;
    __syncthreads();
  }
  SK_STAMP(2);
  // The terms are linear in K: with the prep kernel, slice 0 adds the X term and the whole
  // constant; with in-kernel prep every slice adds its own X term and K_slice * A * B.
  uint32_t cterm = slice == 0 ? p.c0 : 0u;
  if (p.inprep) {
    const uint32_t k_lo = s_begin * kChunkWords * 32u;
    const uint32_t k_hi = min(s_end * kChunkWords * 32u, p.k_logical);
    cterm = (k_hi > k_lo ? k_hi - k_lo : 0u) * (p.coef_w / 2u) * (p.coef_x / 2u);
  }


  // EXT: four accumulators scaled 1, 4, 16, 64 (lo, q4, hi, q64); else lo (+ hi = 16x)
  constexpr bool EXT = SPLIT && N <= 2 && NT <= 2;
  uint32_t lo[NT][4], hi[NT][4], q4[EXT ? NT : 1][4], q64[EXT ? NT : 1][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) lo[nt][e] = hi[nt][e] = 0u;
#pragma unroll
  for (int nt = 0; nt < (EXT ? NT : 1); ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) q4[nt][e] = q64[nt][e] = 0u;

  // B-fragment row of each n-tile for this lane: the feature row, else the zero row, or the
  // all-ones row for the rowsum(U_w) column
  uint32_t xrow[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const uint32_t tok = nt * 8u + g;
    xrow[nt] = tok < p.rows_x ? tok : (tok == ONES ? p.rows_x + 1u : p.rows_x);
  }
  uint32_t cs_slot = 0, phase_bits = 0;
  uint32_t rsa = 0, rsb = 0;  // PR: this thread's share of rowsum(U_w) of rows g, g + 8
  for (uint32_t ti = 0; ti < my_tiles; ++ti) {
    const uint32_t tile = j0 + ti * gs;
    for (uint32_t c = 0; c < cpw; ++c) {
      __syncwarp();  // every lane is done with the slot the next issue overwrites
      issue();
      const uint32_t chunk = s_begin + c * warps_k + wk;
      if (chunk < s_end) {
        if (!p.inprep) apmm_ptx::mbar_wait(&xbars[div_small(chunk - s_begin, p.inv_xpc)], 0);
        apmm_ptx::mbar_wait(&bars[cs_slot], (phase_bits >> cs_slot) & 1u);
        phase_bits ^= 1u << cs_slot;
        if (ti == 0 && c == 0) SK_STAMP(3);  // the first item's weights are in
        // slot layout (TMA box {16 words, 16 rows, planes}): [plane][row][16 words]
        const uint8_t* slot = smem + p.ring_off + (warp * kStages + cs_slot) * SLOT + g * 64u + t * 16u;
        uint4 wa[N], wb[N];
#pragma unroll
        for (int pl = 0; pl < N; ++pl) {
          const bool live = SPLIT || uint32_t(pl) < p.n_planes;
          wa[pl] = live ? *reinterpret_cast<const uint4*>(slot + pl * 1024) : make_uint4(0, 0, 0, 0);
          wb[pl] = live ? *reinterpret_cast<const uint4*>(slot + pl * 1024 + 512) : make_uint4(0, 0, 0, 0);
        }
        if (PR) {
#pragma unroll
          for (int pl = 0; pl < N; ++pl) {
            rsa += (__popc(wa[pl].x) + __popc(wa[pl].y) + __popc(wa[pl].z) + __popc(wa[pl].w)) << pl;
            rsb += (__popc(wb[pl].x) + __popc(wb[pl].y) + __popc(wb[pl].z) + __popc(wb[pl].w)) << pl;
          }
        }
        const uint4* xchunk = reinterpret_cast<const uint4*>(xs + (chunk - s_begin) * xchunk_bytes);
        const uint32_t m4 = frag_rows(p.rows_x) * 4u;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint32_t xa[8], xb[8], ca[8], cb[8];
#pragma unroll
          for (int pl = 0; pl < 8; ++pl) {
            if (pl < N) {
              const uint4& A = wa[pl < N ? pl : 0];
              const uint4& B = wb[pl < N ? pl : 0];
              xa[pl] = w == 0 ? A.x : w == 1 ? A.y : w == 2 ? A.z : A.w;
              xb[pl] = w == 0 ? B.x : w == 1 ? B.y : w == 2 ? B.z : B.w;
            } else {
              xa[pl] = xb[pl] = 0u;
            }
          }
          codes_of_word<N, SPLIT, EXT>(xa, ca, p);
          codes_of_word<N, SPLIT, EXT>(xb, cb, p);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const uint4 x0 = xchunk[(w * 2u + 0u) * m4 + xrow[nt] * 4u + t];
            const uint4 x1 = xchunk[(w * 2u + 1u) * m4 + xrow[nt] * 4u + t];
            if (EXT) {
              mma_u8(lo[nt], ca[0], cb[0], ca[1], cb[1], x0.x, x0.y);
              mma_u8(q4[EXT ? nt : 0], ca[2], cb[2], ca[3], cb[3], x0.z, x0.w);
              mma_u8(hi[nt], ca[4], cb[4], ca[5], cb[5], x1.x, x1.y);
              mma_u8(q64[EXT ? nt : 0], ca[6], cb[6], ca[7], cb[7], x1.z, x1.w);
              continue;
            }
            mma_u8(lo[nt], ca[0], cb[0], ca[1], cb[1], x0.x, x0.y);
            mma_u8(lo[nt], ca[2], cb[2], ca[3], cb[3], x0.z, x0.w);
            if (SPLIT) {
              mma_u8(hi[nt], ca[4], cb[4], ca[5], cb[5], x1.x, x1.y);
              mma_u8(hi[nt], ca[6], cb[6], ca[7], cb[7], x1.z, x1.w);
            } else {
              mma_u8(lo[nt], ca[4], cb[4], ca[5], cb[5], x1.x, x1.y);
              mma_u8(lo[nt], ca[6], cb[6], ca[7], cb[7], x1.z, x1.w);
            }
          }
        }
      }
      cs_slot = cs_slot + 1u == kStages ? 0u : cs_slot + 1u;
    }
    if (ti == 0) SK_STAMP(4);

    // ---------------- end of tile: combine the K groups, epilogue ----------------
    if (ti + 1 == my_tiles) apmm_ptx::pdl_trigger();  // last tile: the next call may start
    {
      uint32_t* mine = red + (wr * 16u) * M_PAD;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const uint32_t c = nt * 8u + 2u * t;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t v = lo[nt][e] + (SPLIT ? (hi[nt][e] >> 4) : 0u);
          if (EXT) {  // exact: the host admits EXT only when 64 K A B < 2^32
            v += (q4[EXT ? nt : 0][e] >> 2) + (q64[EXT ? nt : 0][e] >> 6);
            q4[EXT ? nt : 0][e] = q64[EXT ? nt : 0][e] = 0u;
          }
          atomicAdd(mine + (g + (e >= 2 ? 8u : 0u)) * M_PAD + c + (e & 1), v);
          lo[nt][e] = hi[nt][e] = 0u;
        }
      }
      if (PR) {  // the four t lanes of a row hold different words of it
        rsa += __shfl_xor_sync(0xffffffffu, rsa, 1);
        rsa += __shfl_xor_sync(0xffffffffu, rsa, 2);
        rsb += __shfl_xor_sync(0xffffffffu, rsb, 1);
        rsb += __shfl_xor_sync(0xffffffffu, rsb, 2);
        if (t == 0) {
          atomicAdd(&rsw_s[wr * 16u + g], rsa);
          atomicAdd(&rsw_s[wr * 16u + g + 8u], rsb);
        }
        rsa = rsb = 0u;
      }
    }
    __syncthreads();
    const uint32_t elems = tile_rows * M_PAD;
    for (uint32_t e = tid; e < elems; e += THREADS) {
      const uint32_t rl = e / M_PAD, tok = e % M_PAD;
      const uint32_t row = tile * tile_rows + rl;
      if (row >= p.rows_w || tok >= p.rows_x) continue;
      const uint32_t rsw = PR ? rsw_s[rl] : red[rl * M_PAD + (PR ? 0u : ONES)];
      const uint32_t v = 4u * red[e] - p.coef_w * rsw - p.coef_x * rsx_s[tok] + cterm;
      if (p.slices > 1) {
        atomicAdd(p.acc + (uint64_t(tile) * tile_rows + rl) * M_PAD + tok, v);
        continue;
      }
      const uint64_t o = uint64_t(row) * p.rows_x + tok;
      if (p.yf) {
        const double sw = p.gran_w ? p.s_w[row] : p.s_w[0];
        const double sx = p.gran_x ? p.s_x[tok] : p.s_x[0];
        p.yf[o] = static_cast<float>(__dmul_rn(__dmul_rn(double(int32_t(v)), sw), sx));
      } else {
        p.y[o] = static_cast<int32_t>(v);
      }
    }
    if (p.slices == 1 && ti + 1 == my_tiles) break;  // last tile: red is not reused
    __syncthreads();  // every reader of red is done
    for (uint32_t e = tid; e < elems; e += THREADS) red[e] = 0u;
    if (PR) for (uint32_t q = tid; q < tile_rows; q += THREADS) rsw_s[q] = 0u;
    if (p.slices > 1 && tid == 0) {
      __threadfence();
      const uint32_t prev = atomicAdd(p.counters + tile, 1u);
      s_last = (prev == p.slices - 1) ? 1u : 0u;
    }
    __syncthreads();  // red zeroed before the next tile's adds; s_last visible
    if (p.slices > 1 && s_last) {  // the last slice of this tile: finalise, re-zero
      __threadfence();
      for (uint32_t e = tid; e < elems; e += THREADS) {
        const uint32_t rl = e / M_PAD, tok = e % M_PAD;
        const uint32_t row = tile * tile_rows + rl;
        if (row >= p.rows_w || tok >= p.rows_x) continue;
        uint32_t* ap = p.acc + (uint64_t(tile) * tile_rows + rl) * M_PAD + tok;
        const uint32_t yv = __ldcg(ap);
        const uint64_t o = uint64_t(row) * p.rows_x + tok;
        if (p.yf) {
          const double sw = p.gran_w ? p.s_w[row] : p.s_w[0];
          const double sx = p.gran_x ? p.s_x[tok] : p.s_x[0];
          p.yf[o] = static_cast<float>(__dmul_rn(__dmul_rn(double(int32_t(yv)), sw), sx));
        } else {
          p.y[o] = static_cast<int32_t>(yv);
        }
        __stcg(ap, 0u);
      }
      if (tid == 0) p.counters[tile] = 0u;
    }
    // s_last is next written after the next tile's first barrier
  }
  if (my_tiles == 0) apmm_ptx::pdl_trigger();
  SK_STAMP(5);
}

template <int N, int NT, bool SPLIT, bool PR>
cudaError_t launch_t(const CUtensorMap& tm, const SkinnyParams& p, unsigned grid, uint32_t smem,
                     cudaStream_t s) {
  auto kern = skinny_kernel<N, NT, SPLIT, PR>;
  static DeviceBits attr_set;  // one per instantiation
  const int dev = current_device();
  cudaError_t e;
  if (!attr_set.test(dev)) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sk_smem_budget(N, NT)));
    if (e != cudaSuccess) return e;
    attr_set.set(dev);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(sk_threads(N, NT));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tm, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Kernel variants: SPLIT for n_w <= 4 (N = n_w exactly); otherwise the full transpose with
// N = 4 (n_w <= 4) or N = 8 (n_w 5..8), unused planes masked at run time.
int kernel_n(int n_w, bool split) { return split ? n_w : (n_w <= 4 ? 4 : 8); }

template <int NT, bool PR>
cudaError_t dispatch_np(int n_w, bool split, const CUtensorMap& tm, const SkinnyParams& p,
                        unsigned grid, uint32_t smem, cudaStream_t s) {
  if (split) {
    switch (n_w) {
      case 1: return launch_t<1, NT, true, PR>(tm, p, grid, smem, s);
      case 2: return launch_t<2, NT, true, PR>(tm, p, grid, smem, s);
      case 3: return launch_t<3, NT, true, PR>(tm, p, grid, smem, s);
      default: return launch_t<4, NT, true, PR>(tm, p, grid, smem, s);
    }
  }
  return n_w <= 4 ? launch_t<4, NT, false, PR>(tm, p, grid, smem, s)
                  : launch_t<8, NT, false, PR>(tm, p, grid, smem, s);
}
template <int NT>
cudaError_t dispatch_n(int n_w, bool split, bool pr, const CUtensorMap& tm, const SkinnyParams& p,
                       unsigned grid, uint32_t smem, cudaStream_t s) {
  if constexpr (NT <= 2) {
    if (pr) return dispatch_np<NT, true>(n_w, split, tm, p, grid, smem, s);
  }
  return dispatch_np<NT, false>(n_w, split, tm, p, grid, smem, s);
}

struct Plan {
  uint32_t r, s, slice_chunks, n_tiles, grid, smem, ring_off, red_off;
};

// Work plan: R (16-row groups per tile), S (K slices), grid. The cost counts a warp's
// critical path in item steps (one item = 16 rows x 512 columns): the compute,
// ceil(tiles / CTAs per slice) * (ceil(slice_chunks / warps_k) + epilogue), plus memory
// round trips, ~3 steps per item beyond the one in flight, plus the split-K atomics. The X
// slice, the ring and the reduction buffer share the CTA's shared memory.
Plan plan_for(uint64_t rows_w, uint64_t rows_x, uint32_t chunks, int n, int nt, int num_sms) {
  const uint32_t warps = static_cast<uint32_t>(sk_threads(n, nt) / 32);
  const uint32_t stage_all = warps * slot_bytes(n);  // one ring stage of every warp
  const uint32_t budget = sk_smem_budget(n, nt);
  const uint32_t ctas = static_cast<uint32_t>(num_sms * sk_ctas_per_sm(n, nt));
  Plan best{};
  double best_cost = 1e30;
  static const int force_r = [] {  // dev: APMM_SK_RS="R,S" pins the plan (A/B of the cost model)
    const char* e = APMM_DEV_ENV("APMM_SK_RS");
    return e ? std::atoi(e) : 0;
  }();
  static const int force_s = [] {
    const char* e = APMM_DEV_ENV("APMM_SK_RS");
    const char* c = e ? std::strchr(e, ',') : nullptr;
    return c ? std::atoi(c + 1) : 0;
  }();
  for (uint32_t r = 1; r <= 8 && r <= warps; r <<= 1) {
    if (force_r && r != static_cast<uint32_t>(force_r)) continue;
    const uint32_t warps_k = warps / r;
    const uint64_t n_tiles = (rows_w + 16 * r - 1) / (16 * r);
    for (uint32_t s = 1; s <= chunks; ++s) {
      const uint32_t sc = (chunks + s - 1) / s;
      if ((chunks + sc - 1) / sc != s) continue;  // same plan as a smaller s
      if (force_s && s != static_cast<uint32_t>(force_s)) continue;
      const uint32_t used = sc * chunk_bytes_m(frag_rows(static_cast<uint32_t>(rows_x))) + red_bytes(nt, r);
      if (used + kStages * stage_all + 1024u > budget) continue;  // 1 KB: ring alignment
      const uint32_t per_slice = ctas / s;
      if (per_slice == 0) break;
      const uint64_t gs = n_tiles < per_slice ? n_tiles : per_slice;
      const uint64_t rounds = (n_tiles + gs - 1) / gs;
      const uint32_t cpw = (sc + warps_k - 1) / warps_k;
      const double trips = static_cast<double>(rounds * cpw);
      const double cost = static_cast<double>(rounds) * (cpw + 0.6) + 3.0 * trips +
                          (s > 1 ? 0.25 * rounds + 1.0 : 0.0);
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        best.r = r;
        best.s = s;
        best.slice_chunks = sc;
        best.n_tiles = static_cast<uint32_t>(n_tiles);
        best.grid = static_cast<uint32_t>(gs * s);
      }
    }
  }
  best.ring_off = best.slice_chunks * chunk_bytes_m(frag_rows(static_cast<uint32_t>(rows_x)));
  best.ring_off = (best.ring_off + 1023u) & ~1023u;
  best.red_off = best.ring_off + kStages * stage_all;
  best.smem = best.red_off + red_bytes(nt, best.r);
  return best;
}

// rowsum(U_w) by popcount when the feature rows fill whole n-tiles (8 or 16 rows); otherwise
// through the all-ones feature column
bool popc_rowsum(uint64_t rows_x) { return rows_x % 8 == 0 && rows_x <= 16; }
uint32_t nt_of(uint64_t rows_x) {
  return static_cast<uint32_t>(popc_rowsum(rows_x) ? rows_x / 8 : rows_x / 8 + 1);  // + ones column
}
bool needs_repack(uint64_t k, const void* w) {
  return ((k + 31) / 32) % 4 != 0 || reinterpret_cast<uintptr_t>(w) % 16 != 0;
}
uint64_t frag_half_bytes(uint64_t rows_x, uint64_t k) {
  const uint64_t wpr = (k + 31) / 32;
  const uint64_t chunks = (wpr + kChunkWords - 1) / kChunkWords;
  const uint64_t prep_blocks = (chunks * kChunkWords + kPrepThreads - 1) / kPrepThreads;
  return round_up(chunks * chunk_bytes_m(frag_rows(static_cast<uint32_t>(rows_x))) +
                  rows_x * prep_blocks * 4, 256);
}

}  // namespace

int skinny_launches(uint64_t rows_x) { return rows_x <= kInprepMaxRows ? 1 : 2; }

size_t skinny_acc_bytes(uint64_t rows_w, uint64_t rows_x) {
  // tiles of 16R rows, R <= 8: rows padded to 128 cover every plan; + tile counters
  const uint64_t rows = (rows_w + 127) / 128 * 128;
  return rows * nt_of(rows_x) * 8 * 4 + (rows / 16 + 1) * 4;
}

size_t skinny_scratch_bytes(uint64_t rows_w, uint64_t rows_x, uint64_t k, int n_w,
                            const void* w_planes) {
  size_t b = 2 * frag_half_bytes(rows_x, k);
  if (needs_repack(k, w_planes)) b += uint64_t(n_w) * rows_w * round_up((k + 31) / 32, 4) * 4;
  return b;
}

cudaError_t launch_skinny(const SkinnyArgs& a, cudaStream_t s) {
  SkinnyParams p{};
  const uint32_t nt = nt_of(a.rows_x);
  const uint32_t m_pad = nt * 8u;
  p.rows_w = static_cast<uint32_t>(a.rows_w);
  p.rows_x = static_cast<uint32_t>(a.rows_x);
  p.wpr = static_cast<uint32_t>((a.k + 31) / 32);
  p.n_planes = static_cast<uint32_t>(a.n_w);
  p.chunks_total = (p.wpr + kChunkWords - 1) / kChunkWords;
  const uint32_t A = (1u << a.n_w) - 1u, B = (1u << a.n_x) - 1u;
  // SPLIT keeps a 16x accumulator (needs K A B < 2^28); its EXT form for n_w <= 2 and at
  // most 2 n-tiles keeps a 64x one (needs K A B < 2^26)
  const double kab = static_cast<double>(a.k) * A * B;
  const bool ext_shape = a.n_w <= 2 && nt <= 2;
  const bool split = a.n_w <= 4 && kab < (ext_shape ? 67108864.0 : 268435456.0);
  const int kn = kernel_n(a.n_w, split);
  const bool pr = popc_rowsum(a.rows_x);
  static const int inprep_env = [] {
    const char* e = APMM_DEV_ENV("APMM_SK_INPREP");
    return e ? std::atoi(e) : -1;
  }();
  const Plan pl = plan_for(a.rows_w, a.rows_x, p.chunks_total, kn, static_cast<int>(nt), a.num_sms);
  // In-kernel feature prep up to 8 feature rows (two batched load rounds per thread): saves the
  // prep launch and its PDL round trip; 8192^2 W3A8 M=8 12.25 -> 11.78 us, 4096^2 W2A4 M=8
  // 6.17 -> 5.08 us (profiles/r02/r2_k5_inprep2.txt). Beyond that the redundant per-CTA
  // transposes cost more (and rows_x >= 12 goes to K6 when it can).
  const bool inprep = inprep_env >= 0 ? inprep_env != 0 : a.rows_x <= kInprepMaxRows;
  if (pl.grid == 0) return cudaErrorInvalidConfiguration;
  static const bool show = APMM_DEV_ENV("APMM_DEBUG_PLAN") != nullptr;

  // scratch: [half 0 | half 1] feature fragments + rowsum(U_x) parts, then the repack
  uint8_t* scratch = static_cast<uint8_t*>(a.scratch_ws);
  const uint64_t half_bytes = frag_half_bytes(a.rows_x, a.k);
  uint8_t* xfrag = scratch + (a.ws_half ? half_bytes : 0);
  const uint64_t frag_bytes = uint64_t(p.chunks_total) * chunk_bytes_m(frag_rows(p.rows_x));
  int32_t* rsx = reinterpret_cast<int32_t*>(xfrag + frag_bytes);
  const uint32_t prep_blocks = (p.chunks_total * kChunkWords + kPrepThreads - 1) / kPrepThreads;

  // weights: TMA needs 16-byte row pitch and base; otherwise repack (stream-ordered copy)
  const uint32_t* w = a.w_planes;
  uint64_t pitch_words = p.wpr;
  if (needs_repack(a.k, a.w_planes)) {
    pitch_words = round_up(p.wpr, 4);
    uint32_t* rw = reinterpret_cast<uint32_t*>(scratch + 2 * half_bytes);
    const size_t rows = size_t(a.n_w) * a.rows_w;
    cudaError_t e = cudaMemsetAsync(rw, 0, rows * pitch_words * 4, s);
    if (e == cudaSuccess) {
      e = cudaMemcpy2DAsync(rw, pitch_words * 4, a.w_planes, size_t(p.wpr) * 4, size_t(p.wpr) * 4,
                            rows, cudaMemcpyDeviceToDevice, s);
    }
    if (e != cudaSuccess) return e;
    w = rw;
  }
  CUtensorMap tm;
  {
    const uint64_t dims[3] = {p.wpr, a.rows_w, static_cast<uint64_t>(a.n_w)};
    const uint64_t strides[2] = {pitch_words * 4, pitch_words * 4 * a.rows_w};
    const uint32_t box[3] = {static_cast<uint32_t>(kChunkWords), 16u, static_cast<uint32_t>(a.n_w)};
    if (encode_tmap_3d_u32(&tm, w, dims, strides, box) != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  if (show) {
    std::fprintf(stderr, "[apmm skinny] %llux%llux%llu W%dA%d: R=%u S=%u slice_chunks=%u tiles=%u "
                 "grid=%u smem=%u split=%d repack=%d\n", (unsigned long long)a.rows_w,
                 (unsigned long long)a.rows_x, (unsigned long long)a.k, a.n_w, a.n_x, pl.r, pl.s,
                 pl.slice_chunks, pl.n_tiles, pl.grid, pl.smem, int(split),
                 int(needs_repack(a.k, a.w_planes)));
  }
  const uint64_t rows_pad = uint64_t(pl.n_tiles) * 16u * pl.r;
  p.acc = static_cast<uint32_t*>(a.acc_ws);
  p.counters = p.acc + rows_pad * m_pad;
  p.xfrag = xfrag;
  p.x_planes = a.x_planes;
  p.inprep = inprep ? 1u : 0u;
  p.early_w = a.early_w ? 1u : 0u;
  p.n_x = static_cast<uint32_t>(a.n_x);
  p.k_logical = static_cast<uint32_t>(a.k);
  p.rsx = rsx;
  p.rsx_parts = prep_blocks;
  p.rgroups = pl.r;
  p.slices = pl.s;
  {
    const uint32_t warps = static_cast<uint32_t>(sk_threads(kn, static_cast<int>(nt)) / 32);
    uint32_t l = 0;
    while ((1u << (l + 1)) <= pl.r) ++l;  // R is a power of two
    const uint32_t warps_k = warps >> l;
    p.log2_wk = 0;
    while ((1u << (p.log2_wk + 1)) <= warps_k) ++p.log2_wk;
    p.gs = pl.grid / pl.s;
    p.cpw = (pl.slice_chunks + warps_k - 1) / warps_k;
    p.xpc = (pl.slice_chunks + kXPieces - 1) / kXPieces;
    p.inv_slices = inv_small(pl.s);
    p.inv_gs = inv_small(p.gs);
    p.inv_xpc = inv_small(p.xpc);
    p.inv_sw = inv_small(pl.slice_chunks * kChunkWords);
    p.inv_sw_last = inv_small((p.chunks_total - (pl.s - 1) * pl.slice_chunks) * kChunkWords);
  }
  p.slice_chunks = pl.slice_chunks;
  p.n_tiles = pl.n_tiles;
  p.ring_off = pl.ring_off;
  p.red_off = pl.red_off;
  p.y = a.y;
  p.yf = a.yf;
  p.s_w = a.s_w;
  p.s_x = a.s_x;
  p.gran_w = a.gran_w;
  p.gran_x = a.gran_x;
  p.coef_w = 2u * B;
  p.coef_x = 2u * A;
  p.c0 = static_cast<uint32_t>(a.k) * A * B;
  p.m2 = 2u;
  p.m4 = 4u;
  p.m16 = 16u;
  p.neg1 = 0xFFFFFFFFu;
  if (a.trace) p.ts = a.trace;  // dev launch trace (APMM_TRACE)
  static const bool ts_clock = APMM_DEV_ENV("APMM_TRACE_CLOCK") != nullptr;
  p.ts_clock = ts_clock ? 1u : 0u;
  static const uint32_t x_first = APMM_DEV_ENV("APMM_SK_XFIRST") != nullptr ? 1u : 0u;
  p.x_first = x_first;

  if (!inprep) {  // feature prep (same shared-memory carveout as the streaming kernel: no reconfig)
    static DeviceBits carve_set;
    const int dev = current_device();
    if (!carve_set.test(dev)) {
      cudaFuncSetAttribute(prep_x_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      carve_set.set(dev);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(prep_blocks, frag_rows(p.rows_x));
    cfg.blockDim = dim3(kPrepThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, prep_x_kernel, a.x_planes, p.rows_x, p.wpr, a.n_x,
                                       p.chunks_total * kChunkWords, xfrag, rsx,
                                       a.early_x ? 1u : 0u);
    if (e != cudaSuccess) return e;
  }
  if (a.ev_start) cudaEventRecordWithFlags(a.ev_start, s, a.ev_flags);
  cudaError_t res;
  switch (nt) {
    case 1: res = dispatch_n<1>(a.n_w, split, pr, tm, p, pl.grid, pl.smem, s); break;
    case 2: res = dispatch_n<2>(a.n_w, split, pr, tm, p, pl.grid, pl.smem, s); break;
    case 3: res = dispatch_n<3>(a.n_w, split, pr, tm, p, pl.grid, pl.smem, s); break;
    case 4: res = dispatch_n<4>(a.n_w, split, pr, tm, p, pl.grid, pl.smem, s); break;
    case 5: res = dispatch_n<5>(a.n_w, split, pr, tm, p, pl.grid, pl.smem, s); break;
    case 6: res = dispatch_n<6>(a.n_w, split, pr, tm, p, pl.grid, pl.smem, s); break;
    case 7: res = dispatch_n<7>(a.n_w, split, pr, tm, p, pl.grid, pl.smem, s); break;
    default: res = dispatch_n<8>(a.n_w, split, pr, tm, p, pl.grid, pl.smem, s); break;
  }
  if (a.ev_stop) cudaEventRecordWithFlags(a.ev_stop, s, a.ev_flags);
  return res;
}

}  // namespace apmm_b200
