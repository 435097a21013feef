/*
 * apmm_oracle.c -- TEST INFRASTRUCTURE ONLY (see apmm_oracle.h).
 *
 * A plain-C restatement of the reference's CPU path, written from the reference's
 * documented behaviour. Each function cites the reference file:line (relative to
 * /root/reference/proj) whose semantics it reproduces. Used as the checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg -- never by the product.
 */
#include "apmm_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "../include/apmm_cuda.h"

/* ---------------------------------------------------------------- mt19937_64 ---- */
/* The reference's Rng draws from std::mt19937_64 (include/apmm/rng.hpp:13-16); these
 * are the standard's parameters (C++ [rand.predef]: w=64 n=312 m=156 r=31 ...). */
enum { MT_N = 312, MT_M = 156 };
static const uint64_t MT_A = 0xB5026F5AA96619E9ull;
static const uint64_t MT_UPPER = 0xFFFFFFFF80000000ull;
static const uint64_t MT_LOWER = 0x7FFFFFFFull;

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  r->idx = MT_N;
}

static void mt_twist(orc_rng* r) {
  for (int i = 0; i < MT_N; ++i) {
    const uint64_t y = (r->mt[i] & MT_UPPER) | (r->mt[(i + 1) % MT_N] & MT_LOWER);
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ull) ? MT_A : 0ull);
  }
  r->idx = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

uint64_t orc_rng_below(orc_rng* r, uint64_t n) { return orc_rng_next(r) % n; }

uint64_t orc_rng_range(orc_rng* r, uint64_t lo, uint64_t hi) {
  return lo + orc_rng_below(r, hi - lo + 1);
}

double orc_rng_uniform(orc_rng* r, double lo, double hi) {
  const double unit = (double)(orc_rng_next(r) >> 11) * 0x1.0p-53;
  return lo + unit * (hi - lo);
}

void orc_random_codes(orc_rng* r, uint64_t rows, uint64_t cols, int n, uint8_t* codes) {
  const uint64_t count = 1ull << n;
  for (uint64_t e = 0; e < rows * cols; ++e) codes[e] = (uint8_t)orc_rng_below(r, count);
}

void orc_rng_fill(orc_rng* r, uint64_t count, uint64_t* out) {
  for (uint64_t e = 0; e < count; ++e) out[e] = orc_rng_next(r);
}

/* ----------------------------------------------------------- bipolar format ---- */
static int max_value(int n) { return (1 << n) - 1; }

int orc_decode(unsigned bits, int n) { return 2 * (int)bits - max_value(n); }

int orc_encode(int value, int n, unsigned* bits) {
  if (n < 1 || n > 8) return APMM_E_OUT_OF_RANGE;
  if (value % 2 == 0) return APMM_E_EVEN_VALUE;
  if (abs(value) > max_value(n)) return APMM_E_OUT_OF_RANGE;
  *bits = (unsigned)(value + max_value(n)) / 2u;
  return APMM_OK;
}

/* round_to_grid (bipolar.cpp:63-68): nearest odd integer, ties at even integers go up. */
static int round_to_grid(double t, int maxv) {
  const double q = 2.0 * floor(t / 2.0) + 1.0;
  if (q > maxv) return maxv;
  if (q < -maxv) return -maxv;
  return (int)q;
}

int orc_quantize(const double* x, uint64_t rows, uint64_t cols, int n, int granularity,
                 uint8_t* codes, double* scales) {
  if (n < 1 || n > 8) return APMM_E_OUT_OF_RANGE;
  if (rows == 0 || cols == 0) return APMM_E_DIMENSION_MISMATCH;
  for (uint64_t e = 0; e < rows * cols; ++e) {
    if (!isfinite(x[e])) return APMM_E_NON_FINITE; /* bipolar.cpp:73-75 */
  }
  const int maxv = max_value(n);
  const uint64_t groups = granularity == APMM_PER_ROW ? rows : 1;
  const uint64_t glen = granularity == APMM_PER_ROW ? cols : rows * cols;
  for (uint64_t g = 0; g < groups; ++g) {
    const double* src = x + g * glen;
    double amax = 0.0;
    for (uint64_t i = 0; i < glen; ++i) {
      const double a = fabs(src[i]);
      if (amax < a) amax = a;
    }
    const double s = amax == 0.0 ? 1.0 : amax / (double)maxv; /* bipolar.cpp:91 */
    scales[g] = s;
    for (uint64_t i = 0; i < glen; ++i) {
      const int q = round_to_grid(src[i] / s, maxv);
      codes[g * glen + i] = (uint8_t)((q + maxv) / 2);
    }
  }
  return APMM_OK;
}

void orc_dequantize(const uint8_t* codes, uint64_t rows, uint64_t cols, int n,
                    int granularity, const double* scales, double* out) {
  for (uint64_t r = 0; r < rows; ++r) {
    const double s = granularity == APMM_PER_ROW ? scales[r] : scales[0];
    for (uint64_t c = 0; c < cols; ++c) {
      out[r * cols + c] = s * orc_decode(codes[r * cols + c], n);
    }
  }
}

/* --------------------------------------------------------------- bit planes ---- */
static uint64_t wpr_of(uint64_t cols) { return (cols + 31) / 32; }

void orc_pack(const uint8_t* codes, uint64_t rows, uint64_t cols, int n, uint32_t* planes) {
  const uint64_t wpr = wpr_of(cols);
  memset(planes, 0, sizeof(uint32_t) * (size_t)n * rows * wpr);
  for (uint64_t r = 0; r < rows; ++r) {
    for (uint64_t k = 0; k < cols; ++k) {
      const unsigned c = codes[r * cols + k];
      for (int p = 0; p < n; ++p) {
        planes[((uint64_t)p * rows + r) * wpr + (k >> 5)] |= ((c >> p) & 1u) << (k & 31);
      }
    }
  }
}

void orc_unpack(const uint32_t* planes, uint64_t rows, uint64_t cols, int n, uint8_t* codes) {
  const uint64_t wpr = wpr_of(cols);
  for (uint64_t r = 0; r < rows; ++r) {
    for (uint64_t k = 0; k < cols; ++k) {
      unsigned c = 0;
      for (int p = 0; p < n; ++p) {
        c |= ((planes[((uint64_t)p * rows + r) * wpr + (k >> 5)] >> (k & 31)) & 1u) << p;
      }
      codes[r * cols + k] = (uint8_t)c;
    }
  }
}

int orc_check_padding(const uint32_t* planes, uint64_t rows, uint64_t cols, int n) {
  const unsigned tail = (unsigned)(cols & 31);
  if (tail == 0) return APMM_OK;
  const uint32_t pad = ~((1u << tail) - 1u);
  const uint64_t wpr = wpr_of(cols);
  for (uint64_t pr = 0; pr < (uint64_t)n * rows; ++pr) {
    if (planes[(pr + 1) * wpr - 1] & pad) return APMM_E_OUT_OF_RANGE;
  }
  return APMM_OK;
}

/* ------------------------------------------------------------ plane products ---- */
static int64_t xor_popc(const uint32_t* a, const uint32_t* b, uint64_t words) {
  int64_t total = 0;
  uint64_t i = 0;
  for (; i + 2 <= words; i += 2) {
    uint64_t va, vb;
    memcpy(&va, a + i, 8);
    memcpy(&vb, b + i, 8);
    total += __builtin_popcountll(va ^ vb);
  }
  if (i < words) total += __builtin_popcount(a[i] ^ b[i]);
  return total;
}

int orc_dot_1bit_xor(const uint32_t* a, uint64_t a_words, const uint32_t* b,
                     uint64_t b_words, uint64_t k, int64_t* out) {
  if (k == 0) return APMM_E_OUT_OF_RANGE;                          /* kernel.cpp:117 */
  const uint64_t need = wpr_of(k);
  if (a_words != need || b_words != need) return APMM_E_LENGTH_MISMATCH; /* :118-121 */
  *out = (int64_t)k - 2 * xor_popc(a, b, need);
  return APMM_OK;
}

int orc_plane_products(const uint32_t* w, uint64_t rows_w, int n_w, const uint32_t* x,
                       uint64_t rows_x, int n_x, uint64_t k, int32_t* stack) {
  const uint64_t wpr = wpr_of(k);
  for (int i = 0; i < n_w; ++i) {
    for (int j = 0; j < n_x; ++j) {
      int32_t* out = stack + (uint64_t)(i * n_x + j) * rows_w * rows_x;
      for (uint64_t m = 0; m < rows_w; ++m) {
        const uint32_t* wr = w + ((uint64_t)i * rows_w + m) * wpr;
        for (uint64_t n = 0; n < rows_x; ++n) {
          const uint32_t* xr = x + ((uint64_t)j * rows_x + n) * wpr;
          out[m * rows_x + n] = (int32_t)((int64_t)k - 2 * xor_popc(wr, xr, wpr));
        }
      }
    }
  }
  return APMM_OK;
}

int orc_recover(const int32_t* stack, int n_w, int n_x, uint64_t m, uint64_t n, int32_t* y) {
  for (uint64_t e = 0; e < m * n; ++e) {
    int64_t acc = 0;
    for (int i = 0; i < n_w; ++i) {
      for (int j = 0; j < n_x; ++j) {
        acc += ((int64_t)1 << (i + j)) * stack[(uint64_t)(i * n_x + j) * m * n + e];
      }
    }
    if (acc > INT32_MAX || acc < INT32_MIN) return APMM_E_OVERFLOW; /* kernel.cpp:174-177 */
    y[e] = (int32_t)acc;
  }
  return APMM_OK;
}

int64_t orc_overflow_bound(int n_w, int n_x, uint64_t k) {
  return (int64_t)k * max_value(n_w) * max_value(n_x);
}

/* ------------------------------------------------------------------ matmul_ap ---- */
typedef struct {
  const uint32_t* w;
  const uint32_t* x;
  uint64_t rows_w, rows_x, k, wpr;
  int n_w, n_x;
  uint64_t b_m, b_n, chunk_words;
  uint64_t m_begin, m_end;
  int32_t* y;
} ap_job;

/* One contiguous block of output rows, tiled exactly as kernel.cpp:214-251: per tile,
 * per K chunk, per weight plane i, per (m, n): feature-side recovery over j first
 * (sum_j dot << j), then one weight-side shift (<< i) into the int32 tile. */
static void ap_rows(const ap_job* jb) {
  const uint64_t tile_cap = jb->b_m * jb->b_n;
  int32_t* tile = (int32_t*)malloc(sizeof(int32_t) * (size_t)tile_cap);
  const uint64_t xps = jb->rows_x * jb->wpr; /* feature plane stride */
  for (uint64_t m0 = jb->m_begin; m0 < jb->m_end; m0 += jb->b_m) {
    const uint64_t tm = (jb->m_end - m0) < jb->b_m ? (jb->m_end - m0) : jb->b_m;
    for (uint64_t n0 = 0; n0 < jb->rows_x; n0 += jb->b_n) {
      const uint64_t tn = (jb->rows_x - n0) < jb->b_n ? (jb->rows_x - n0) : jb->b_n;
      memset(tile, 0, sizeof(int32_t) * (size_t)(tm * tn));
      for (uint64_t w0 = 0; w0 < jb->wpr; w0 += jb->chunk_words) {
        const uint64_t cw = (jb->wpr - w0) < jb->chunk_words ? (jb->wpr - w0) : jb->chunk_words;
        const uint64_t end_bits = (w0 + cw) * 32 < jb->k ? (w0 + cw) * 32 : jb->k;
        const int64_t chunk_bits = (int64_t)(end_bits - w0 * 32);
        for (int i = 0; i < jb->n_w; ++i) {
          for (uint64_t mt = 0; mt < tm; ++mt) {
            const uint32_t* wr = jb->w + ((uint64_t)i * jb->rows_w + m0 + mt) * jb->wpr + w0;
            for (uint64_t nt = 0; nt < tn; ++nt) {
              const uint32_t* xr = jb->x + (n0 + nt) * jb->wpr + w0;
              int64_t part = 0;
              for (int j = 0; j < jb->n_x; ++j) {
                part += (chunk_bits - 2 * xor_popc(wr, xr + (uint64_t)j * xps, cw)) << j;
              }
              tile[mt * tn + nt] += (int32_t)(part << i);
            }
          }
        }
      }
      for (uint64_t mt = 0; mt < tm; ++mt) {
        memcpy(jb->y + (m0 + mt) * jb->rows_x + n0, tile + mt * tn, sizeof(int32_t) * tn);
      }
    }
  }
  free(tile);
}

static int ap_validate(int n_w, int n_x, uint64_t rows_w, uint64_t rows_x, uint64_t k) {
  if (n_w < 1 || n_w > 8 || n_x < 1 || n_x > 8) return APMM_E_OUT_OF_RANGE;
  if (rows_w == 0 || rows_x == 0 || k == 0) return APMM_E_DIMENSION_MISMATCH;
  if (orc_overflow_bound(n_w, n_x, k) > INT32_MAX) return APMM_E_OVERFLOW_BOUND;
  return APMM_OK;
}

int orc_matmul_ap(const uint32_t* w, uint64_t rows_w, int n_w, const uint32_t* x,
                  uint64_t rows_x, int n_x, uint64_t k, uint64_t b_m, uint64_t b_n,
                  uint64_t b_k, int32_t* y) {
  if (b_m == 0 || b_n == 0 || b_k < 32 || b_k % 32 != 0) return APMM_E_OUT_OF_RANGE;
  const int st = ap_validate(n_w, n_x, rows_w, rows_x, k);
  if (st != APMM_OK) return st;
  ap_job jb = {w, x, rows_w, rows_x, k, wpr_of(k), n_w, n_x, b_m, b_n, b_k / 32, 0, rows_w, y};
  ap_rows(&jb);
  return APMM_OK;
}

static void* ap_thread(void* arg) {
  ap_rows((const ap_job*)arg);
  return NULL;
}

int orc_matmul_ap_mt(const uint32_t* w, uint64_t rows_w, int n_w, const uint32_t* x,
                     uint64_t rows_x, int n_x, uint64_t k, int threads, int32_t* y) {
  const int st = ap_validate(n_w, n_x, rows_w, rows_x, k);
  if (st != APMM_OK) return st;
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > rows_w) threads = (int)rows_w;
  ap_job* jobs = (ap_job*)calloc((size_t)threads, sizeof(ap_job));
  pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    ap_job jb = {w, x, rows_w, rows_x, k, wpr_of(k), n_w, n_x, 64, 64, 16,
                 rows_w * (uint64_t)t / (uint64_t)threads,
                 rows_w * (uint64_t)(t + 1) / (uint64_t)threads, y};
    jobs[t] = jb;
    pthread_create(&tids[t], NULL, ap_thread, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
  free(jobs);
  free(tids);
  return APMM_OK;
}

/* ---------------------------------------------------------------- naive oracle ---- */
int orc_naive_matmul(const int32_t* a, uint64_t m, const int32_t* b_kmajor, uint64_t n,
                     uint64_t k, int32_t* y) {
  for (uint64_t r = 0; r < m; ++r) {
    for (uint64_t c = 0; c < n; ++c) {
      int64_t acc = 0;
      for (uint64_t e = 0; e < k; ++e) acc += (int64_t)a[r * k + e] * b_kmajor[c * k + e];
      if (acc > INT32_MAX || acc < INT32_MIN) return APMM_E_OVERFLOW; /* oracle.cpp:20-23 */
      y[r * n + c] = (int32_t)acc;
    }
  }
  return APMM_OK;
}

int orc_decoded_matmul(const uint8_t* w_codes, uint64_t rows_w, int n_w,
                       const uint8_t* x_codes, uint64_t rows_x, int n_x, uint64_t k,
                       int32_t* y) {
  int32_t* a = (int32_t*)malloc(sizeof(int32_t) * (size_t)(rows_w * k));
  int32_t* b = (int32_t*)malloc(sizeof(int32_t) * (size_t)(rows_x * k));
  for (uint64_t e = 0; e < rows_w * k; ++e) a[e] = orc_decode(w_codes[e], n_w);
  for (uint64_t e = 0; e < rows_x * k; ++e) b[e] = orc_decode(x_codes[e], n_x);
  const int st = orc_naive_matmul(a, rows_w, b, rows_x, k, y);
  free(a);
  free(b);
  return st;
}

void orc_dequant_epilogue(const int32_t* y, uint64_t rows, uint64_t cols,
                          const double* w_scales, int w_gran, const double* x_scales,
                          int x_gran, float* out) {
  for (uint64_t m = 0; m < rows; ++m) {
    const double sw = w_gran == APMM_PER_ROW ? w_scales[m] : w_scales[0];
    for (uint64_t n = 0; n < cols; ++n) {
      const double sx = x_gran == APMM_PER_ROW ? x_scales[n] : x_scales[0];
      out[m * cols + n] = (float)((double)y[m * cols + n] * sw * sx);
    }
  }
}
