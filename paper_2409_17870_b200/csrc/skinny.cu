// skinny.cu -- K5: the WnAm bipolar-INT GEMM for few feature rows (decode / small-M LLM
// shapes), HBM-bound on the packed weight planes.
//
// Why a separate kernel. With M_tok <= 64 the GEMM does ~2*M ops per weight code, so the
// roofline is the HBM read of the packed weight planes (n_w bits per weight). The large-M
// path (expand -> u8 codes in HBM -> tcgen05 GEMM) would write and re-read 8/n_w times
// those bytes. Here the weight planes go from HBM straight into registers (128-bit
// non-allocating loads), are turned into u8 code fragments in registers by a partial 8x8
// bit transpose, and feed legacy-pipe mma.sync m16n8k32 u8 x u8 -> s32 MMAs. Tensor-core
// throughput is irrelevant at this M; what matters is the ALU cost per weight code, which
// the transpose keeps at ~0.7 ops/code for n_w <= 4 (see below).
//
// The algebra is the same as the large-M path: one u8 x u8 MMA
// of the unsigned codes performs the whole 2^(i+j)-weighted plane-pair recovery of the
// reference's matmul_ap (kernel.cpp:187-254); the rank-1 term is applied in the epilogue.
//
// Fragment mapping (PTX m16n8k32 .u8): thread (g = lane/4, t = lane%4) supplies A rows g
// and g+8 and B column g at K slots {4t+b, 16+4t+b}. The K order inside the MMA is free as
// long as A and B agree, and the slot -> column map below depends only on (t, slot), never
// on g:
//   thread t loads plane words [16c + 4t, +4) (128 columns) of its two weight rows;
//   a 32-column word is bit-transposed so that register r, byte B holds column 8B + r;
//   X codes come from the expand kernel in exactly that order (byte 4r+B of a 32-byte
//   group = column 8B + r), so the B fragment of the MMA that uses A registers (r, r+1)
//   is X's group registers (r, r+1).
// For n_w <= 4 only two of the three delta-swap stages run: register r (r < 4) then holds
// column 8B+r in its low nibble and column 8B+4+r in its high nibble. `x & 0x0F0F0F0F`
// gives the first, `x & 0xF0F0F0F0` gives 16x the second; the latter goes into a separate
// accumulator that is divided by 16 at the end (exact: the host admits this variant only
// when K*(2^n_w-1)*(2^n_x-1) < 2^28, so 16x the partial sum fits in 32 bits).
//
// Work split: CTA = 8 warps x 16 weight rows = 128 rows; grid.y splits K into slices of
// whole 512-column chunks. Each CTA stages its X slice in shared memory in per-lane
// fragment order (conflict-free 128-bit reads), accumulates its partial products in
// registers, and adds them into an int32 workspace with wrapping atomics (exact mod 2^32,
// order-independent). The last CTA of a row block (counter) applies the rank-1 recovery
// / dequant epilogue, writes Y, and re-zeroes the workspace for the next call.
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "ptx.cuh"

namespace apmm_b200 {
namespace {

constexpr int kSkThreads = 256;
constexpr int kSkWarps = kSkThreads / 32;
constexpr int kChunkWords = 16;  // 512 columns per warp iteration
constexpr uint32_t kSkSmemMax = 96u * 1024u;  // X slice budget per CTA

struct SkinnyParams {
  const uint32_t* w;         // weight planes, reference layout [n_w][rows_w][wpr]
  const uint8_t* xc;         // feature codes [rows_x][kpad], expand order
  const int32_t* rowsum_x;   // [rows_x]
  uint32_t rows_w, rows_x, wpr, kpad_words;
  uint32_t chunks_total, chunks_per_slice;
  uint32_t* acc;             // [row_blocks * 128][m_pad], zero on entry and on exit
  uint32_t* acc_rs;          // [row_blocks * 128] partial rowsum(U_w)
  uint32_t* counters;        // [row_blocks]
  int32_t* y;
  float* yf;
  const double* s_w;
  const double* s_x;
  int gran_w, gran_x;
  uint32_t coef_w, coef_x, c0;
};

APMM_DEV uint4 ld_stream_v4(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

APMM_DEV void mma_u8(uint32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                     uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

APMM_DEV void swap_sel(uint32_t& a, uint32_t& b, int s, uint32_t m) {
  const uint32_t na = (a & ~(m << s)) | ((b << s) & (m << s));
  b = (b & ~m) | ((a >> s) & m);
  a = na;
}

// Four plane words of one weight row (row = plane index in x[]), for 4 consecutive words.
template <int N>
struct RowWords {
  uint4 p[N];
};

template <int N, bool VEC>
APMM_DEV void load_row(RowWords<N>& r, const uint32_t* base, uint64_t pstride, uint32_t w0,
                       uint32_t wpr, bool row_ok) {
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const uint32_t* p = base + i * pstride;
    if (VEC && row_ok && w0 + 3 < wpr) {
      r.p[i] = ld_stream_v4(p + w0);
    } else {
      r.p[i].x = row_ok && w0 + 0 < wpr ? __ldg(p + w0 + 0) : 0u;
      r.p[i].y = row_ok && w0 + 1 < wpr ? __ldg(p + w0 + 1) : 0u;
      r.p[i].z = row_ok && w0 + 2 < wpr ? __ldg(p + w0 + 2) : 0u;
      r.p[i].w = row_ok && w0 + 3 < wpr ? __ldg(p + w0 + 3) : 0u;
    }
  }
}

template <int N>
APMM_DEV uint32_t word_of(const RowWords<N>& r, int i, int w) {
  return w == 0 ? r.p[i].x : w == 1 ? r.p[i].y : w == 2 ? r.p[i].z : r.p[i].w;
}

// Codes of one 32-column word. SPLIT (N <= 4): lo[r] = codes of columns 8B+r, hi[r] = 16x
// codes of columns 8B+4+r (r < 4). Otherwise full[r] = codes of columns 8B+r (r < 8).
template <int N, bool SPLIT>
APMM_DEV void codes_of_word(const RowWords<N>& rw, int w, uint32_t (&o)[8], int32_t& rowsum) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = i < N ? word_of(rw, i, w) : 0u;
#pragma unroll
  for (int i = 0; i < N; ++i) rowsum += __popc(x[i]) << i;
  if (SPLIT) {
    swap_sel(x[0], x[2], 2, 0x33333333u);
    swap_sel(x[1], x[3], 2, 0x33333333u);
    swap_sel(x[0], x[1], 1, 0x55555555u);
    swap_sel(x[2], x[3], 1, 0x55555555u);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      o[r] = x[r] & 0x0F0F0F0Fu;
      o[4 + r] = x[r] & 0xF0F0F0F0u;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) swap_sel(x[i], x[i + 4], 4, 0x0F0F0F0Fu);
#pragma unroll
    for (int i = 0; i < 8; i += 4) {
      swap_sel(x[i], x[i + 2], 2, 0x33333333u);
      swap_sel(x[i + 1], x[i + 3], 2, 0x33333333u);
    }
#pragma unroll
    for (int i = 0; i < 8; i += 2) swap_sel(x[i], x[i + 1], 1, 0x55555555u);
#pragma unroll
    for (int r = 0; r < 8; ++r) o[r] = x[r];
  }
}

// Shared-memory X layout per 512-column chunk: [w 0..3][nt][half 0..1][lane 0..31] x 16 B.
// Lane (g, t) of n-tile nt, word w, half h holds bytes [16h, 16h+16) of the 32-byte code
// group of feature row nt*8+g, word 16*chunk + 4t + w.
template <int NT>
__host__ __device__ constexpr uint32_t chunk_smem_bytes() {
  return 4u * NT * 2u * 32u * 16u;
}

// Two CTAs per SM where the register budget (128) allows it without spilling.
template <int N, int NT>
constexpr int sk_min_blocks() {
  return (N <= 4 && NT <= 4) ? 2 : 1;
}

template <int N, int NT, bool SPLIT, bool VEC>
__global__ void __launch_bounds__(kSkThreads, sk_min_blocks<N, NT>()) skinny_kernel(const SkinnyParams p) {
  extern __shared__ __align__(16) uint8_t xs[];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t g = lane >> 2, t = lane & 3;
  const uint32_t row_blk = blockIdx.x;
  const uint32_t row_a = row_blk * 128u + warp * 16u + g, row_b = row_a + 8u;
  const bool ok_a = row_a < p.rows_w, ok_b = row_b < p.rows_w;
  const uint32_t c_begin = blockIdx.y * p.chunks_per_slice;
  const uint32_t c_end = min(c_begin + p.chunks_per_slice, p.chunks_total);
  const uint64_t pstride = uint64_t(p.rows_w) * p.wpr;
  const uint32_t* wa = p.w + uint64_t(ok_a ? row_a : 0) * p.wpr;
  const uint32_t* wb = p.w + uint64_t(ok_b ? row_b : 0) * p.wpr;

  // The weight planes are inputs of this call: their first loads may overlap the feature
  // expand kernel still running ahead of us (PDL); the X codes may not.
  RowWords<N> cur_a, cur_b, nxt_a, nxt_b;
  load_row<N, VEC>(cur_a, wa, pstride, c_begin * kChunkWords + 4 * t, p.wpr, ok_a);
  load_row<N, VEC>(cur_b, wb, pstride, c_begin * kChunkWords + 4 * t, p.wpr, ok_b);
  apmm_ptx::pdl_wait();

  // ---- stage the X slice (fragment order) ----
  {
    const uint32_t nchunks = c_end - c_begin;
    const uint32_t pieces = nchunks * (chunk_smem_bytes<NT>() / 16u);
    for (uint32_t q = threadIdx.x; q < pieces; q += kSkThreads) {
      const uint32_t ln = q & 31u, h = (q >> 5) & 1u;
      const uint32_t rest = q >> 6;  // (chunk_local * 4 + w) * NT + nt
      const uint32_t nt = rest % NT, cw = rest / NT;
      const uint32_t w = cw & 3u, cl = cw >> 2;
      const uint32_t tok = nt * 8u + (ln >> 2);
      const uint32_t word = (c_begin + cl) * kChunkWords + 4u * (ln & 3u) + w;
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (tok < p.rows_x && word < p.kpad_words) {
        v = __ldg(reinterpret_cast<const uint4*>(p.xc + uint64_t(tok) * p.kpad_words * 32u +
                                                 uint64_t(word) * 32u + h * 16u));
      }
      reinterpret_cast<uint4*>(xs)[q] = v;
    }
  }
  __syncthreads();

  uint32_t lo[NT][4], hi[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) lo[nt][e] = hi[nt][e] = 0u;
  int32_t rs_a = 0, rs_b = 0;

  const uint4* xs4 = reinterpret_cast<const uint4*>(xs);
  for (uint32_t c = c_begin; c < c_end; ++c) {
    if (c + 1 < c_end) {
      load_row<N, VEC>(nxt_a, wa, pstride, (c + 1) * kChunkWords + 4 * t, p.wpr, ok_a);
      load_row<N, VEC>(nxt_b, wb, pstride, (c + 1) * kChunkWords + 4 * t, p.wpr, ok_b);
    }
    const uint4* xchunk = xs4 + (c - c_begin) * (chunk_smem_bytes<NT>() / 16u);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      uint32_t ca[8], cb[8];
      codes_of_word<N, SPLIT>(cur_a, w, ca, rs_a);
      codes_of_word<N, SPLIT>(cur_b, w, cb, rs_b);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const uint4 x0 = xchunk[((w * NT + nt) * 2 + 0) * 32 + lane];
        const uint4 x1 = xchunk[((w * NT + nt) * 2 + 1) * 32 + lane];
        if (SPLIT) {
          mma_u8(lo[nt], ca[0], cb[0], ca[1], cb[1], x0.x, x0.y);
          mma_u8(lo[nt], ca[2], cb[2], ca[3], cb[3], x0.z, x0.w);
          mma_u8(hi[nt], ca[4], cb[4], ca[5], cb[5], x1.x, x1.y);
          mma_u8(hi[nt], ca[6], cb[6], ca[7], cb[7], x1.z, x1.w);
        } else {
          mma_u8(lo[nt], ca[0], cb[0], ca[1], cb[1], x0.x, x0.y);
          mma_u8(lo[nt], ca[2], cb[2], ca[3], cb[3], x0.z, x0.w);
          mma_u8(lo[nt], ca[4], cb[4], ca[5], cb[5], x1.x, x1.y);
          mma_u8(lo[nt], ca[6], cb[6], ca[7], cb[7], x1.z, x1.w);
        }
      }
    }
    cur_a = nxt_a;
    cur_b = nxt_b;
  }

  // ---- partial sums -> workspace (wrapping adds: exact and order-independent) ----
  const uint32_t m_pad = NT * 8u;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t row = (e < 2) ? row_a : row_b;
      const uint32_t tok = nt * 8u + 2u * t + (e & 1u);
      const uint32_t s = lo[nt][e] + (SPLIT ? (hi[nt][e] >> 4) : 0u);
      atomicAdd(p.acc + uint64_t(row) * m_pad + tok, s);
    }
  }
  rs_a += __shfl_xor_sync(0xffffffffu, rs_a, 1);
  rs_a += __shfl_xor_sync(0xffffffffu, rs_a, 2);
  rs_b += __shfl_xor_sync(0xffffffffu, rs_b, 1);
  rs_b += __shfl_xor_sync(0xffffffffu, rs_b, 2);
  if (t == 0) {
    atomicAdd(p.acc_rs + row_a, static_cast<uint32_t>(rs_a));
    atomicAdd(p.acc_rs + row_b, static_cast<uint32_t>(rs_b));
  }

  // ---- last CTA of this row block: rank-1 recovery / dequant epilogue ----
  __shared__ uint32_t last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(p.counters + row_blk, 1u);
    last = (prev == gridDim.y - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // allow the next call's expand to start (it writes the other workspace half and waits
  // for us before it completes)
  apmm_ptx::pdl_trigger();
  const uint32_t total = 128u * m_pad;
  for (uint32_t i = threadIdx.x; i < total; i += kSkThreads) {
    const uint32_t row = row_blk * 128u + i / m_pad, tok = i % m_pad;
    uint32_t* ap = p.acc + uint64_t(row) * m_pad + tok;
    if (row < p.rows_w && tok < p.rows_x) {
      const uint32_t s = __ldcg(ap);
      const uint32_t rsw = __ldcg(p.acc_rs + row);
      const uint32_t rsx = static_cast<uint32_t>(__ldg(p.rowsum_x + tok));
      const uint32_t v = 4u * s + p.c0 - p.coef_w * rsw - p.coef_x * rsx;
      const uint64_t o = uint64_t(row) * p.rows_x + tok;
      if (p.yf) {
        const double sw = p.gran_w ? p.s_w[row] : p.s_w[0];
        const double sx = p.gran_x ? p.s_x[tok] : p.s_x[0];
        p.yf[o] = static_cast<float>(__dmul_rn(__dmul_rn(double(int32_t(v)), sw), sx));
      } else {
        p.y[o] = static_cast<int32_t>(v);
      }
    }
    __stcg(ap, 0u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 128u; i += kSkThreads) __stcg(p.acc_rs + row_blk * 128u + i, 0u);
  if (threadIdx.x == 0) p.counters[row_blk] = 0u;
}

template <int N, int NT, bool SPLIT, bool VEC>
cudaError_t launch_t(const SkinnyParams& p, dim3 grid, uint32_t smem, cudaStream_t s) {
  auto kern = skinny_kernel<N, NT, SPLIT, VEC>;
  static bool attr_set = false;  // one per instantiation
  cudaError_t e;
  if (!attr_set) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSkSmemMax));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kSkThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, p);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int NT, bool SPLIT, bool VEC>
cudaError_t dispatch_n(int n, const SkinnyParams& p, dim3 grid, uint32_t smem, cudaStream_t s) {
  if constexpr (SPLIT) {
    switch (n) {
      case 1: return launch_t<1, NT, SPLIT, VEC>(p, grid, smem, s);
      case 2: return launch_t<2, NT, SPLIT, VEC>(p, grid, smem, s);
      case 3: return launch_t<3, NT, SPLIT, VEC>(p, grid, smem, s);
      default: return launch_t<4, NT, SPLIT, VEC>(p, grid, smem, s);
    }
  } else {
  switch (n) {
    case 1: case 2: case 3: case 4: return launch_t<4, NT, false, VEC>(p, grid, smem, s);
    case 5: return launch_t<5, NT, false, VEC>(p, grid, smem, s);
    case 6: return launch_t<6, NT, false, VEC>(p, grid, smem, s);
    case 7: return launch_t<7, NT, false, VEC>(p, grid, smem, s);
    default: return launch_t<8, NT, false, VEC>(p, grid, smem, s);
  }
  }
}

template <int NT>
cudaError_t dispatch_nt(int n, bool split, bool vec, const SkinnyParams& p, dim3 grid,
                        uint32_t smem, cudaStream_t s) {
  if (split) {
    return vec ? dispatch_n<NT, true, true>(n, p, grid, smem, s)
               : dispatch_n<NT, true, false>(n, p, grid, smem, s);
  }
  return vec ? dispatch_n<NT, false, true>(n, p, grid, smem, s)
             : dispatch_n<NT, false, false>(n, p, grid, smem, s);
}

}  // namespace

uint32_t skinny_m_pad(uint64_t rows_x) {
  const uint32_t nt = rows_x <= 8 ? 1u : rows_x <= 16 ? 2u : rows_x <= 32 ? 4u : 8u;
  return nt * 8u;
}

size_t skinny_ws_bytes(uint64_t rows_w, uint64_t rows_x) {
  const uint64_t blocks = (rows_w + 127) / 128;
  return blocks * 128 * skinny_m_pad(rows_x) * 4 + blocks * 128 * 4 + blocks * 4;
}

cudaError_t launch_skinny(const SkinnyArgs& a, cudaStream_t s) {
  SkinnyParams p{};
  const uint32_t m_pad = skinny_m_pad(a.rows_x);
  const int nt = static_cast<int>(m_pad / 8);
  const uint64_t blocks = (a.rows_w + 127) / 128;
  p.w = a.w_planes;
  p.xc = a.codes_x;
  p.rowsum_x = a.rowsum_x;
  p.rows_w = static_cast<uint32_t>(a.rows_w);
  p.rows_x = static_cast<uint32_t>(a.rows_x);
  p.wpr = static_cast<uint32_t>((a.k + 31) / 32);
  p.kpad_words = static_cast<uint32_t>(a.kpad / 32);
  p.chunks_total = (p.wpr + kChunkWords - 1) / kChunkWords;
  // K slices: enough CTAs for ~2 per SM, but no more X restaging than needed, and the X
  // slice must fit the shared-memory budget.
  const uint32_t per_chunk = 4u * nt * 2u * 32u * 16u;
  const uint32_t max_chunks_smem = kSkSmemMax / per_chunk;
  const uint64_t want_ctas = 2ull * static_cast<uint64_t>(a.num_sms);
  uint64_t slices = (want_ctas + blocks - 1) / blocks;
  if (slices < 1) slices = 1;
  if (slices > p.chunks_total) slices = p.chunks_total;
  uint32_t cps = static_cast<uint32_t>((p.chunks_total + slices - 1) / slices);
  if (cps > max_chunks_smem) cps = max_chunks_smem;
  if (cps < 1) cps = 1;
  p.chunks_per_slice = cps;
  const uint32_t nslices = (p.chunks_total + cps - 1) / cps;
  uint8_t* ws = static_cast<uint8_t*>(a.ws);
  p.acc = reinterpret_cast<uint32_t*>(ws);
  p.acc_rs = reinterpret_cast<uint32_t*>(ws + blocks * 128 * m_pad * 4);
  p.counters = reinterpret_cast<uint32_t*>(ws + blocks * 128 * m_pad * 4 + blocks * 128 * 4);
  p.y = a.y;
  p.yf = a.yf;
  p.s_w = a.s_w;
  p.s_x = a.s_x;
  p.gran_w = a.gran_w;
  p.gran_x = a.gran_x;
  const uint32_t A = (1u << a.n_w) - 1u, B = (1u << a.n_x) - 1u;
  p.coef_w = 2u * B;
  p.coef_x = 2u * A;
  p.c0 = static_cast<uint32_t>(a.k) * A * B;
  const bool split = a.n_w <= 4 && static_cast<double>(a.k) * A * B < 268435456.0;
  const bool vec = (p.wpr % 4u) == 0u && (reinterpret_cast<uintptr_t>(a.w_planes) % 16u) == 0u;
  const dim3 grid(static_cast<unsigned>(blocks), nslices);
  const uint32_t smem = cps * per_chunk;
  switch (nt) {
    case 1: return dispatch_nt<1>(a.n_w, split, vec, p, grid, smem, s);
    case 2: return dispatch_nt<2>(a.n_w, split, vec, p, grid, smem, s);
    case 4: return dispatch_nt<4>(a.n_w, split, vec, p, grid, smem, s);
    default: return dispatch_nt<8>(a.n_w, split, vec, p, grid, smem, s);
  }
}

}  // namespace apmm_b200
