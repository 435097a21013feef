// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper around the UNMODIFIED reference library, compiled from the
// reference's own sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/libapmm_ref.so by oracle/Makefile. Lets tests/ and bench.py call the
// reference itself (to pin the C restatement in apmm_oracle.c, to generate
// tests/golden/, and as the CPU baseline / `--impl reference` arm). No reference
// source is copied into this repository.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "apmm/bipolar.hpp"
#include "apmm/bitplane.hpp"
#include "apmm/error.hpp"
#include "apmm/kernel.hpp"
#include "apmm/oracle.hpp"
#include "apmm/rng.hpp"
#include "apmm/tensor_file.hpp"
#include "apmm/verify.hpp"

#include "../include/apmm_cuda.h"

using namespace apmm;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const EvenValue*>(&e)) return APMM_E_EVEN_VALUE;
  if (dynamic_cast<const OutOfRange*>(&e)) return APMM_E_OUT_OF_RANGE;
  if (dynamic_cast<const NonFinite*>(&e)) return APMM_E_NON_FINITE;
  if (dynamic_cast<const LengthMismatch*>(&e)) return APMM_E_LENGTH_MISMATCH;
  if (dynamic_cast<const DimensionMismatch*>(&e)) return APMM_E_DIMENSION_MISMATCH;
  if (dynamic_cast<const IndexOutOfBounds*>(&e)) return APMM_E_INDEX_OUT_OF_BOUNDS;
  if (dynamic_cast<const OverflowBound*>(&e)) return APMM_E_OVERFLOW_BOUND;
  if (dynamic_cast<const Overflow*>(&e)) return APMM_E_OVERFLOW;
  if (dynamic_cast<const ParseError*>(&e)) return APMM_E_PARSE;
  if (dynamic_cast<const IoError*>(&e)) return APMM_E_IO;
  return APMM_E_INVALID_ARGUMENT;
}

#define GUARD(body)                          \
  try {                                      \
    body;                                    \
    return APMM_OK;                          \
  } catch (const std::exception& e) {        \
    return status_of(e);                     \
  }

PackedBitPlanes packed(const uint32_t* words, uint64_t rows, uint64_t cols, int n) {
  const uint64_t wpr = (cols + 31) / 32;
  return PackedBitPlanes(rows, cols, BitWidth(n),
                         std::vector<uint32_t>(words, words + uint64_t(n) * rows * wpr));
}

// Rows [r0, r1) of every plane, as a standalone PackedBitPlanes (for row slicing).
PackedBitPlanes row_slice(const uint32_t* words, uint64_t rows, uint64_t cols, int n,
                          uint64_t r0, uint64_t r1) {
  const uint64_t wpr = (cols + 31) / 32;
  std::vector<uint32_t> buf;
  buf.reserve(uint64_t(n) * (r1 - r0) * wpr);
  for (int p = 0; p < n; ++p) {
    const uint32_t* base = words + (uint64_t(p) * rows + r0) * wpr;
    buf.insert(buf.end(), base, base + (r1 - r0) * wpr);
  }
  return PackedBitPlanes(r1 - r0, cols, BitWidth(n), std::move(buf));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Rng stream (rng.hpp) -- to pin the oracle's mt19937_64 restatement.
void ref_rng_draws(uint64_t seed, uint64_t count, uint64_t* out) {
  Rng rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_u64();
}

int ref_quantize(const double* x, uint64_t rows, uint64_t cols, int n, int gran,
                 uint8_t* codes, double* scales) {
  GUARD({
    const QuantizedTensor q =
        quantize(RealMatrix(rows, cols, std::vector<double>(x, x + rows * cols)), BitWidth(n),
                 gran == APMM_PER_ROW ? Granularity::PerRow : Granularity::PerTensor);
    std::memcpy(codes, q.codes().raw_bits().data(), rows * cols);
    std::memcpy(scales, q.scales().data(), q.scales().size() * sizeof(double));
  })
}

int ref_pack(const uint8_t* codes, uint64_t rows, uint64_t cols, int n, uint32_t* words) {
  GUARD({
    const PackedBitPlanes p = decompose_and_pack(
        CodeMatrix(rows, cols, BitWidth(n), std::vector<uint8_t>(codes, codes + rows * cols)));
    std::memcpy(words, p.words().data(), p.words().size() * sizeof(uint32_t));
  })
}

int ref_unpack(const uint32_t* words, uint64_t rows, uint64_t cols, int n, uint8_t* codes) {
  GUARD({
    const CodeMatrix c = unpack(packed(words, rows, cols, n));
    std::memcpy(codes, c.raw_bits().data(), rows * cols);
  })
}

int ref_matmul_ap(const uint32_t* w, uint64_t rows_w, int n_w, const uint32_t* x,
                  uint64_t rows_x, int n_x, uint64_t k, uint64_t b_m, uint64_t b_n,
                  uint64_t b_k, int32_t* y) {
  GUARD({
    const AccumMatrix out = matmul_ap(packed(w, rows_w, k, n_w), packed(x, rows_x, k, n_x),
                                      TileConfig(b_m, b_n, b_k));
    std::memcpy(y, out.data.data(), out.data.size() * sizeof(int32_t));
  })
}

int ref_decoded_matmul(const uint8_t* wc, uint64_t rows_w, int n_w, const uint8_t* xc,
                       uint64_t rows_x, int n_x, uint64_t k, int32_t* y) {
  GUARD({
    const IntMatrix out = decoded_matmul(
        CodeMatrix(rows_w, k, BitWidth(n_w), std::vector<uint8_t>(wc, wc + rows_w * k)),
        CodeMatrix(rows_x, k, BitWidth(n_x), std::vector<uint8_t>(xc, xc + rows_x * k)));
    std::memcpy(y, out.data.data(), out.data.size() * sizeof(int32_t));
  })
}

int ref_plane_products(const uint32_t* w, uint64_t rows_w, int n_w, const uint32_t* x,
                       uint64_t rows_x, int n_x, uint64_t k, int32_t* stack, int32_t* y) {
  GUARD({
    const PlaneProductStack s =
        compute_plane_products(packed(w, rows_w, k, n_w), packed(x, rows_x, k, n_x));
    int32_t* dst = stack;
    for (int i = 0; i < n_w; ++i) {
      for (int j = 0; j < n_x; ++j) {
        const IntMatrix& p = s.product(unsigned(i), unsigned(j));
        std::memcpy(dst, p.data.data(), p.data.size() * sizeof(int32_t));
        dst += p.data.size();
      }
    }
    const AccumMatrix r = recover(s);
    std::memcpy(y, r.data.data(), r.data.size() * sizeof(int32_t));
  })
}

int ref_dot_1bit_xor(const uint32_t* a, uint64_t a_words, const uint32_t* b, uint64_t b_words,
                     uint64_t k, int64_t* out) {
  GUARD({
    *out = dot_1bit_xor(std::span<const uint32_t>(a, a_words),
                        std::span<const uint32_t>(b, b_words), k);
  })
}

// ---- APMM v1 tensor files (tensor_file.cpp): the reference's own serializer / parser ----
// quantize (bipolar.cpp:72-100) -> TensorFile::from_quantized -> serialize_tensor; with
// out == nullptr only *len is set.
int ref_serialize_quantized(const double* x, uint64_t rows, uint64_t cols, int n, int gran,
                            uint8_t* out, uint64_t cap, uint64_t* len) {
  GUARD({
    const QuantizedTensor q =
        quantize(RealMatrix(rows, cols, std::vector<double>(x, x + rows * cols)), BitWidth(n),
                 gran == APMM_PER_ROW ? Granularity::PerRow : Granularity::PerTensor);
    const std::vector<uint8_t> b = serialize_tensor(TensorFile::from_quantized(q));
    *len = b.size();
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  })
}

// RealMatrix -> TensorFile::from_real (f32) -> serialize_tensor.
int ref_serialize_float(const double* x, uint64_t rows, uint64_t cols, uint8_t* out, uint64_t cap,
                        uint64_t* len) {
  GUARD({
    const std::vector<uint8_t> b = serialize_tensor(
        TensorFile::from_real(RealMatrix(rows, cols, std::vector<double>(x, x + rows * cols))));
    *len = b.size();
    if (out && cap >= b.size()) std::memcpy(out, b.data(), b.size());
  })
}

// parse_tensor + to_packed (quantized) -> words, scales; status as the reference throws.
int ref_parse_to_packed(const uint8_t* bytes, uint64_t n, uint32_t* words, double* scales) {
  GUARD({
    const TensorFile t = parse_tensor(std::span<const uint8_t>(bytes, n));
    const PackedBitPlanes p = t.to_packed();
    std::memcpy(words, p.words().data(), p.words().size() * sizeof(uint32_t));
    std::memcpy(scales, t.scales.data(), t.scales.size() * sizeof(double));
  })
}

// ---- CPU baseline: the reference's matmul_ap, row-sliced over std::threads --------
// (SPEC.md:266 permits parallel tiles). Packing/slicing is done in prepare (excluded
// from timing, like apmm.cpp:163-172); run() times exactly the matmul_ap calls.
struct RefJob {
  std::vector<PackedBitPlanes> w_slices;
  std::vector<uint64_t> row_begin;
  std::unique_ptr<PackedBitPlanes> x;
  std::vector<AccumMatrix> out;
  uint64_t rows_w = 0, rows_x = 0;
};

void* ref_job_prepare(const uint32_t* w, uint64_t rows_w, int n_w, const uint32_t* x,
                      uint64_t rows_x, int n_x, uint64_t k, int threads) {
  try {
    auto* job = new RefJob();
    job->rows_w = rows_w;
    job->rows_x = rows_x;
    threads = std::max(1, std::min<int>(threads, int(rows_w)));
    for (int t = 0; t < threads; ++t) {
      const uint64_t r0 = rows_w * uint64_t(t) / uint64_t(threads);
      const uint64_t r1 = rows_w * uint64_t(t + 1) / uint64_t(threads);
      job->w_slices.push_back(row_slice(w, rows_w, k, n_w, r0, r1));
      job->row_begin.push_back(r0);
    }
    job->x = std::make_unique<PackedBitPlanes>(packed(x, rows_x, k, n_x));
    job->out.resize(job->w_slices.size());
    return job;
  } catch (const std::exception& e) {
    status_of(e);
    return nullptr;
  }
}

// Runs every slice once (all threads), returns wall seconds.
double ref_job_run(void* handle) {
  auto* job = static_cast<RefJob*>(handle);
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (size_t t = 0; t < job->w_slices.size(); ++t) {
    pool.emplace_back([job, t] { job->out[t] = matmul_ap(job->w_slices[t], *job->x); });
  }
  for (auto& th : pool) th.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void ref_job_result(void* handle, int32_t* y) {
  auto* job = static_cast<RefJob*>(handle);
  for (size_t t = 0; t < job->out.size(); ++t) {
    const AccumMatrix& o = job->out[t];
    std::memcpy(y + job->row_begin[t] * job->rows_x, o.data.data(),
                o.data.size() * sizeof(int32_t));
  }
}

void ref_job_free(void* handle) { delete static_cast<RefJob*>(handle); }

// ---- run_verify with the default (reference) kernel --------------------------------
// Returns the number of properties; writes pass flags; first failure detail via
// ref_last_error().
int ref_run_verify(uint64_t seed, int cases, uint64_t max_dim, uint64_t max_k, int* passed,
                   int max_props) {
  try {
    VerifyOptions opt;
    opt.seed = seed;
    opt.cases = cases;
    opt.max_dim = max_dim;
    opt.max_k = max_k;
    const VerifyReport rep = run_verify(opt);
    g_err.clear();
    int i = 0;
    for (const auto& p : rep.properties) {
      if (i < max_props) passed[i] = p.passed ? 1 : 0;
      if (!p.passed && g_err.empty()) g_err = p.name + ": " + p.detail;
      ++i;
    }
    return i;
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

}  // extern "C"
