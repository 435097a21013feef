// apmm_b200.hpp -- header-only C++ drop-in for the reference's hot path.
//
// Include this next to the reference's own headers (proj/include) and call
// apmm::b200::matmul_ap / decompose_and_pack / unpack / quantize with the reference's own
// types; or hand apmm::b200::kernel_fn() to apmm::run_verify (the KernelFn seam,
// verify.hpp:23-24). Everything runs on the B200 through the C ABI in apmm_cuda.h
// (link -lapmm_b200); failures are rethrown as the reference's apmm::Error subclasses
// (error.hpp:9-70), with the same validation order as the reference.
//
// Only the PUBLIC interface of the reference types is used, so this adapter compiles
// against an unmodified reference tree.
#pragma once

#include <algorithm>
#include <cstdint>
#include <filesystem>
#include <span>
#include <string>
#include <vector>

#include "apmm/bipolar.hpp"
#include "apmm/bitplane.hpp"
#include "apmm/error.hpp"
#include "apmm/kernel.hpp"
#include "apmm/matrix.hpp"
#include "apmm/tensor_file.hpp"
#include "apmm/verify.hpp"
#include "apmm_cuda.h"

namespace apmm::b200 {

[[noreturn]] inline void throw_status(int st) {
  const std::string msg = std::string("B200: ") + apmm_last_error();
  switch (st) {
    case APMM_E_EVEN_VALUE: throw EvenValue(msg);
    case APMM_E_OUT_OF_RANGE: throw OutOfRange(msg);
    case APMM_E_NON_FINITE: throw NonFinite(msg);
    case APMM_E_LENGTH_MISMATCH: throw LengthMismatch(msg);
    case APMM_E_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case APMM_E_INDEX_OUT_OF_BOUNDS: throw IndexOutOfBounds(msg);
    case APMM_E_OVERFLOW: throw Overflow(msg);
    case APMM_E_OVERFLOW_BOUND: throw OverflowBound(msg);
    case APMM_E_PARSE: throw ParseError(msg);
    case APMM_E_IO: throw IoError(msg);
    default: throw Error(msg);
  }
}

inline void check(int st) {
  if (st != APMM_OK) throw_status(st);
}

// One context per thread and device (contexts are not thread-safe).
class Device {
 public:
  explicit Device(int device = 0) { check(apmm_ctx_create(&ctx_, device)); }
  ~Device() { apmm_ctx_destroy(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  apmm_ctx* get() const { return ctx_; }

 private:
  apmm_ctx* ctx_ = nullptr;
};

inline Device& default_device() {
  thread_local Device dev(0);
  return dev;
}

// kernel.hpp:86-87 -- same contract, computed by the sm_100a tensor-core kernel.
inline AccumMatrix matmul_ap(const PackedBitPlanes& weights, const PackedBitPlanes& features,
                             const TileConfig& /*schedule only*/ = {}) {
  if (weights.logical_cols() != features.logical_cols()) {  // kernel.cpp:189-192
    throw DimensionMismatch("operands disagree on K: " + std::to_string(weights.logical_cols()) +
                            " vs " + std::to_string(features.logical_cols()));
  }
  AccumMatrix out(weights.logical_rows(), features.logical_rows());
  check(apmm_matmul_ap(default_device().get(), weights.words().data(), weights.logical_rows(),
                       weights.width().n(), features.words().data(), features.logical_rows(),
                       features.width().n(), weights.logical_cols(), out.data.data()));
  return out;
}

// kernel.hpp:61-62 -- k - 2 popc(a ^ b); OutOfRange for k == 0, LengthMismatch unless both
// spans hold exactly ceil(k/32) words (kernel.cpp:117-121).
inline std::int64_t dot_1bit_xor(std::span<const std::uint32_t> a,
                                 std::span<const std::uint32_t> b, std::size_t k_logical) {
  std::int64_t out = 0;
  check(apmm_dot_1bit_xor(default_device().get(), a.data(), a.size(), b.data(), b.size(),
                          k_logical, &out));
  return out;
}

// kernel.hpp:66-67 -- one plane pair as a 1-bit x 1-bit GEMM on the device.
inline IntMatrix matmul_plane_pair(const PackedBitPlanes& weights, unsigned weight_plane,
                                   const PackedBitPlanes& features, unsigned feature_plane) {
  if (weights.logical_cols() != features.logical_cols()) {  // kernel.cpp:127-130
    throw DimensionMismatch("operands disagree on K: " + std::to_string(weights.logical_cols()) +
                            " vs " + std::to_string(features.logical_cols()));
  }
  IntMatrix out(weights.logical_rows(), features.logical_rows());
  check(apmm_matmul_plane_pair(default_device().get(), weights.words().data(),
                               weights.logical_rows(), weights.width().n(),
                               static_cast<int>(weight_plane), features.words().data(),
                               features.logical_rows(), features.width().n(),
                               static_cast<int>(feature_plane), weights.logical_cols(),
                               out.data.data()));
  return out;
}

// kernel.hpp:70-71 -- every plane pair, each a 1-bit x 1-bit GEMM on the device.
inline PlaneProductStack compute_plane_products(const PackedBitPlanes& weights,
                                                const PackedBitPlanes& features) {
  if (weights.logical_cols() != features.logical_cols()) {
    throw DimensionMismatch("operands disagree on K: " + std::to_string(weights.logical_cols()) +
                            " vs " + std::to_string(features.logical_cols()));
  }
  const int nw = weights.width().n(), nx = features.width().n();
  const std::size_t m = weights.logical_rows(), n = features.logical_rows();
  std::vector<std::int32_t> flat(static_cast<std::size_t>(nw) * nx * m * n);
  check(apmm_compute_plane_products(default_device().get(), weights.words().data(), m, nw,
                                    features.words().data(), n, nx, weights.logical_cols(),
                                    flat.data()));
  std::vector<IntMatrix> products;
  products.reserve(static_cast<std::size_t>(nw) * nx);
  for (std::size_t p = 0; p < static_cast<std::size_t>(nw) * nx; ++p) {
    IntMatrix mat(m, n);
    std::copy(flat.begin() + p * m * n, flat.begin() + (p + 1) * m * n, mat.data.begin());
    products.push_back(std::move(mat));
  }
  return {weights.width(), features.width(), weights.logical_cols(), std::move(products)};
}

// kernel.hpp:74 -- shift-and-add recovery on the device (int64, checked narrowing).
inline AccumMatrix recover(const PlaneProductStack& stack) {
  const int nw = stack.weight_width().n(), nx = stack.feature_width().n();
  const std::size_t m = stack.rows(), n = stack.cols();
  std::vector<std::int32_t> flat(static_cast<std::size_t>(nw) * nx * m * n);
  for (int i = 0; i < nw; ++i) {
    for (int j = 0; j < nx; ++j) {
      const IntMatrix& p = stack.product(static_cast<unsigned>(i), static_cast<unsigned>(j));
      std::copy(p.data.begin(), p.data.end(),
                flat.begin() + (static_cast<std::size_t>(i) * nx + j) * m * n);
    }
  }
  AccumMatrix out(m, n);
  check(apmm_recover(default_device().get(), flat.data(), nw, nx, stack.k_logical(), m, n,
                     out.data.data()));
  return out;
}

// verify.hpp:23-24 -- plug the GPU into the reference's property suite.
inline KernelFn kernel_fn() {
  return [](const PackedBitPlanes& w, const PackedBitPlanes& x, const TileConfig& cfg) {
    return ::apmm::b200::matmul_ap(w, x, cfg);
  };
}

// bitplane.hpp:49
inline PackedBitPlanes decompose_and_pack(const CodeMatrix& codes) {
  const std::size_t words =
      static_cast<std::size_t>(codes.width().n()) * codes.rows() * ((codes.cols() + 31) / 32);
  std::vector<std::uint32_t> buf(words);
  check(apmm_decompose_and_pack(default_device().get(), codes.raw_bits().data(), codes.rows(),
                                codes.cols(), codes.width().n(), buf.data()));
  return PackedBitPlanes(codes.rows(), codes.cols(), codes.width(), std::move(buf));
}

// bitplane.hpp:52
inline CodeMatrix unpack(const PackedBitPlanes& packed) {
  std::vector<std::uint8_t> bits(packed.logical_rows() * packed.logical_cols());
  check(apmm_unpack(default_device().get(), packed.words().data(), packed.logical_rows(),
                    packed.logical_cols(), packed.width().n(), bits.data()));
  return CodeMatrix(packed.logical_rows(), packed.logical_cols(), packed.width(), std::move(bits));
}

// bipolar.hpp:130 (fp64, bit-identical codes and scales)
inline QuantizedTensor quantize(const RealMatrix& values, BitWidth width, Granularity gran) {
  const int g = gran == Granularity::PerRow ? APMM_PER_ROW : APMM_PER_TENSOR;
  std::vector<std::uint8_t> bits(values.rows * values.cols);
  std::vector<std::uint32_t> planes(static_cast<std::size_t>(width.n()) * values.rows *
                                    ((values.cols + 31) / 32));
  std::vector<double> scales(g == APMM_PER_ROW ? values.rows : 1);
  check(apmm_quantize_pack(default_device().get(), values.data.data(), values.rows, values.cols,
                           width.n(), g, bits.data(), planes.data(), scales.data()));
  return QuantizedTensor(CodeMatrix(values.rows, values.cols, width, std::move(bits)), gran,
                         std::move(scales));
}

// matmul_ap + the CLI dequant epilogue (tools/apmm.cpp:329-340) fused on the device.
inline RealMatrix matmul_ap_dequant(const PackedBitPlanes& weights, const std::vector<double>& w_scales,
                                    Granularity w_gran, const PackedBitPlanes& features,
                                    const std::vector<double>& x_scales, Granularity x_gran) {
  if (weights.logical_cols() != features.logical_cols()) {
    throw DimensionMismatch("operands disagree on K");
  }
  std::vector<float> out(weights.logical_rows() * features.logical_rows());
  check(apmm_matmul_ap_dequant(
      default_device().get(), weights.words().data(), weights.logical_rows(), weights.width().n(),
      w_scales.data(), w_gran == Granularity::PerRow ? APMM_PER_ROW : APMM_PER_TENSOR,
      features.words().data(), features.logical_rows(), features.width().n(), x_scales.data(),
      x_gran == Granularity::PerRow ? APMM_PER_ROW : APMM_PER_TENSOR, weights.logical_cols(),
      out.data()));
  RealMatrix real(weights.logical_rows(), features.logical_rows());
  for (std::size_t e = 0; e < out.size(); ++e) real.data[e] = out[e];
  return real;
}

// tensor_file.hpp:61 + to_packed (tensor_file.cpp:124-130): parse a reference APMM v1
// file straight into DEVICE buffers (planes in the PackedBitPlanes layout, scales; or a
// float tensor widened to f64). Sizes from the returned header; buffers may be null.
inline apmm_tensor_info load_tensor_file_to_device(const std::filesystem::path& path,
                                                   std::uint32_t* dev_planes, double* dev_scales,
                                                   double* dev_values) {
  apmm_tensor_info info{};
  check(apmm_tensor_file_load(default_device().get(), path.string().c_str(), &info, dev_planes,
                              dev_scales, dev_values));
  return info;
}

}  // namespace apmm::b200
