"""Python mirror of the reference's public C++ API (proj/include/apmm/*.hpp) on top of the
B200 C ABI (include/apmm_cuda.h, libapmm_b200.so).

Names, argument meaning and error classes follow the reference so code written against
it reads the same:

=====================================  ====================================================
reference (C++)                        here
=====================================  ====================================================
apmm::BitWidth (bipolar.hpp:14-32)     BitWidth
apmm::Granularity (bipolar.hpp:100)    Granularity
apmm::TileConfig (kernel.hpp:14-30)    TileConfig (validated; schedule-only, results never
                                       depend on it -- SPEC.md:252)
apmm::PackedBitPlanes (bitplane.hpp)   PackedBitPlanes (numpy u32 buffer, same layout)
apmm::quantize (bipolar.hpp:130)       quantize -> QuantizedTensor
apmm::decompose_and_pack / unpack      decompose_and_pack / unpack
apmm::overflow_bound (kernel.hpp:78)   overflow_bound
apmm::matmul_ap (kernel.hpp:86)        matmul_ap -> numpy int32 [rows_w, rows_x]
CLI dequant epilogue (apmm.cpp:329)    matmul_ap_dequant -> numpy float32
apmm::Error hierarchy (error.hpp)      Error, EvenValue, OutOfRange, ... (same names)
=====================================  ====================================================

All compute runs on the GPU through the C ABI; there is no CPU fallback. Device-pointer
variants (``cu_*``) take torch CUDA tensors and enqueue on torch's current stream.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib


# ---- errors (error.hpp:9-70) -------------------------------------------------------------
class Error(RuntimeError):
    """Base class, apmm::Error."""


class EvenValue(Error): pass
class OutOfRange(Error): pass
class NonFinite(Error): pass
class LengthMismatch(Error): pass
class DimensionMismatch(Error): pass
class IndexOutOfBounds(Error): pass
class Overflow(Error): pass
class OverflowBound(Error): pass
class InvalidArgument(Error): pass
class CudaError(Error): pass
class NoDevice(Error): pass
class UnsupportedDevice(Error): pass


_STATUS_TO_ERROR = {
    1: EvenValue, 2: OutOfRange, 3: NonFinite, 4: LengthMismatch, 5: DimensionMismatch,
    6: IndexOutOfBounds, 7: Overflow, 8: OverflowBound, 9: InvalidArgument, 100: CudaError,
    101: NoDevice, 102: UnsupportedDevice,
}


def _check(status: int) -> None:
    if status != 0:
        lib = _lib.load()
        msg = lib.apmm_last_error().decode(errors="replace")
        raise _STATUS_TO_ERROR.get(status, Error)(msg)


# ---- value types ---------------------------------------------------------------------------
class BitWidth:
    """bipolar.hpp:14-32 -- widths in [1, 8]."""

    __slots__ = ("_n",)

    def __init__(self, n: int):
        if not (1 <= int(n) <= 8):
            raise OutOfRange("bit width must be in [1, 8]")
        self._n = int(n)

    def n(self) -> int:
        return self._n

    def max_value(self) -> int:
        return (1 << self._n) - 1

    def code_count(self) -> int:
        return 1 << self._n

    def __eq__(self, other) -> bool:
        return isinstance(other, BitWidth) and other._n == self._n

    def __repr__(self) -> str:
        return f"BitWidth({self._n})"


class Granularity(enum.IntEnum):
    PerTensor = 0
    PerRow = 1


@dataclass(frozen=True)
class TileConfig:
    """kernel.hpp:14-30 / kernel.cpp:69-77. Schedule-only: the GPU path accepts and
    validates it, and its results are identical for every valid configuration."""

    block_rows: int = 64
    block_cols: int = 64
    block_k_bits: int = 512

    def __post_init__(self):
        if self.block_rows == 0 or self.block_cols == 0:
            raise OutOfRange("tile dimensions must be positive")
        if self.block_k_bits < 32 or self.block_k_bits % 32 != 0:
            raise OutOfRange("b_k must be a positive multiple of 32 bits")


def words_per_row(cols: int) -> int:
    return (int(cols) + 31) // 32


class PackedBitPlanes:
    """bitplane.hpp:19-45: n planes, plane-major, row, ceil(cols/32) u32 words, LSB-first,
    zero padding (validated on construction exactly like bitplane.cpp:7-33)."""

    def __init__(self, logical_rows: int, logical_cols: int, width: BitWidth, buffer):
        if logical_rows == 0 or logical_cols == 0:
            raise DimensionMismatch("PackedBitPlanes dimensions must be positive")
        self._rows, self._cols, self._width = int(logical_rows), int(logical_cols), width
        self._wpr = words_per_row(logical_cols)
        buf = np.ascontiguousarray(buffer, dtype=np.uint32).reshape(-1)
        expected = width.n() * self._rows * self._wpr
        if buf.size != expected:
            raise LengthMismatch(f"packed buffer holds {buf.size} words, expected {expected}")
        tail = self._cols & 31
        if tail:
            pad = np.uint32(~((1 << tail) - 1) & 0xFFFFFFFF)
            last = buf.reshape(width.n() * self._rows, self._wpr)[:, -1]
            if np.any(last & pad):
                raise OutOfRange("packed buffer has nonzero padding bits")
        self._buf = buf

    def logical_rows(self) -> int:
        return self._rows

    def logical_cols(self) -> int:
        return self._cols

    def width(self) -> BitWidth:
        return self._width

    def words_per_row(self) -> int:
        return self._wpr

    def words(self) -> np.ndarray:
        return self._buf

    def plane_row(self, plane: int, row: int) -> np.ndarray:
        if plane >= self._width.n():
            raise IndexOutOfBounds(f"plane {plane} out of range for width {self._width.n()}")
        if row >= self._rows:
            raise IndexOutOfBounds(f"row {row} out of range for {self._rows} rows")
        off = (plane * self._rows + row) * self._wpr
        return self._buf[off:off + self._wpr]

    def __eq__(self, other) -> bool:
        return (isinstance(other, PackedBitPlanes) and self._rows == other._rows
                and self._cols == other._cols and self._width == other._width
                and np.array_equal(self._buf, other._buf))


@dataclass
class QuantizedTensor:
    """bipolar.hpp:106-127: codes (u8 [rows, cols]) + granularity + fp64 scales, plus the
    packed planes the GPU quantizer produced in the same pass."""

    codes: np.ndarray
    width: BitWidth
    granularity: Granularity
    scales: np.ndarray
    packed: PackedBitPlanes

    def scale_for_row(self, r: int) -> float:
        return float(self.scales[0] if self.granularity == Granularity.PerTensor else self.scales[r])


# ---- device context -------------------------------------------------------------------------
class Context:
    """Owns an apmm_ctx (one device, private stream, reusable workspace)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        _check(self.lib.apmm_ctx_create(C.byref(h), int(device)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.apmm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launch_count(self) -> int:
        return int(self.lib.apmm_ctx_launch_count(self.h))

    def enable_timing(self, enable: bool = True) -> None:
        _check(self.lib.apmm_ctx_enable_timing(self.h, int(bool(enable))))

    def kernel_time(self, kernel: int = 0):
        """(total device ms, launches) of kernel class 0=GEMM / 1=expand since last call."""
        ms, n = C.c_double(), C.c_uint64()
        _check(self.lib.apmm_ctx_kernel_time(self.h, int(kernel), C.byref(ms), C.byref(n)))
        return ms.value, int(n.value)


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def version() -> str:
    return _lib.load().apmm_version().decode()


# ---- host API (mirrors the reference one for one) -------------------------------------------
def overflow_bound(weight_width: BitWidth, feature_width: BitWidth, k: int) -> int:
    """kernel.cpp:183-185."""
    out = C.c_int64()
    _check(_lib.load().apmm_overflow_bound(weight_width.n(), feature_width.n(), int(k),
                                           C.byref(out)))
    return out.value


def decompose_and_pack(codes: np.ndarray, width: BitWidth, ctx: Context | None = None
                       ) -> PackedBitPlanes:
    """bitplane.cpp:48-66 on the GPU (codes: u8 [rows, cols], each < 2^n)."""
    ctx = ctx or default_context()
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    if codes.ndim != 2:
        raise DimensionMismatch("codes must be a 2-D matrix")
    rows, cols = codes.shape
    out = np.empty(width.n() * rows * words_per_row(cols), dtype=np.uint32)
    _check(ctx.lib.apmm_decompose_and_pack(ctx.h, _ptr(codes), rows, cols, width.n(), _ptr(out)))
    return PackedBitPlanes(rows, cols, width, out)


def unpack(packed: PackedBitPlanes, ctx: Context | None = None) -> np.ndarray:
    """bitplane.cpp:68-84 on the GPU."""
    ctx = ctx or default_context()
    out = np.empty((packed.logical_rows(), packed.logical_cols()), dtype=np.uint8)
    _check(ctx.lib.apmm_unpack(ctx.h, _ptr(packed.words()), packed.logical_rows(),
                               packed.logical_cols(), packed.width().n(), _ptr(out)))
    return out


def quantize(values: np.ndarray, width: BitWidth, granularity: Granularity,
             ctx: Context | None = None) -> QuantizedTensor:
    """bipolar.cpp:72-100 (fp64, bit-identical codes and scales) fused with the pack."""
    ctx = ctx or default_context()
    x = np.ascontiguousarray(values, dtype=np.float64)
    if x.ndim != 2:
        raise DimensionMismatch("values must be a 2-D matrix")
    rows, cols = x.shape
    codes = np.empty((rows, cols), dtype=np.uint8)
    planes = np.empty(width.n() * rows * words_per_row(cols), dtype=np.uint32)
    scales = np.empty(rows if granularity == Granularity.PerRow else 1, dtype=np.float64)
    _check(ctx.lib.apmm_quantize_pack(ctx.h, _ptr(x), rows, cols, width.n(), int(granularity),
                                      _ptr(codes), _ptr(planes), _ptr(scales)))
    return QuantizedTensor(codes, width, Granularity(granularity), scales,
                           PackedBitPlanes(rows, cols, width, planes))


def matmul_ap(weights: PackedBitPlanes, features: PackedBitPlanes,
              config: TileConfig = TileConfig(), ctx: Context | None = None) -> np.ndarray:
    """kernel.cpp:187-254 on the GPU: int32 [weights.rows, features.rows], bit-exact."""
    ctx = ctx or default_context()
    if weights.logical_cols() != features.logical_cols():
        raise DimensionMismatch(f"operands disagree on K: {weights.logical_cols()} vs "
                                f"{features.logical_cols()}")
    y = np.empty((weights.logical_rows(), features.logical_rows()), dtype=np.int32)
    _check(ctx.lib.apmm_matmul_ap(ctx.h, _ptr(weights.words()), weights.logical_rows(),
                                  weights.width().n(), _ptr(features.words()),
                                  features.logical_rows(), features.width().n(),
                                  weights.logical_cols(), _ptr(y)))
    return y


class PlaneProductStack:
    """kernel.hpp:36-56 / kernel.cpp:79-113: the n_w*n_x plane-pair products of one
    multiplication, entry [i, j] = weight plane i x feature plane j, each in [-K, K]."""

    def __init__(self, weight_width: BitWidth, feature_width: BitWidth, k_logical: int,
                 products: np.ndarray):
        products = np.ascontiguousarray(products, dtype=np.int32)
        if products.ndim != 4 or products.shape[:2] != (weight_width.n(), feature_width.n()):
            raise LengthMismatch(f"expected {weight_width.n() * feature_width.n()} plane products")
        self._ww, self._fw, self._k, self._p = weight_width, feature_width, int(k_logical), products

    def weight_width(self) -> BitWidth:
        return self._ww

    def feature_width(self) -> BitWidth:
        return self._fw

    def k_logical(self) -> int:
        return self._k

    def rows(self) -> int:
        return self._p.shape[2]

    def cols(self) -> int:
        return self._p.shape[3]

    def product(self, weight_plane: int, feature_plane: int) -> np.ndarray:
        if not (0 <= weight_plane < self._ww.n() and 0 <= feature_plane < self._fw.n()):
            raise IndexOutOfBounds(f"plane pair ({weight_plane}, {feature_plane}) out of range")
        return self._p[weight_plane, feature_plane]

    def products(self) -> np.ndarray:
        return self._p


def matmul_plane_pair(weights: PackedBitPlanes, weight_plane: int, features: PackedBitPlanes,
                      feature_plane: int, ctx: Context | None = None) -> np.ndarray:
    """kernel.cpp:125-144 on the GPU: XOR dots of one weight plane against one feature plane."""
    ctx = ctx or default_context()
    if weights.logical_cols() != features.logical_cols():
        raise DimensionMismatch(f"operands disagree on K: {weights.logical_cols()} vs "
                                f"{features.logical_cols()}")
    import torch
    k = weights.logical_cols()
    dev = torch.device("cuda", ctx.device)
    w = torch.from_numpy(weights.words().view(np.int32)).to(dev)
    x = torch.from_numpy(features.words().view(np.int32)).to(dev)
    y = torch.empty((weights.logical_rows(), features.logical_rows()), dtype=torch.int32, device=dev)
    _check(ctx.lib.apmm_cu_matmul_plane_pair(
        ctx.h, C.c_void_p(w.data_ptr()), weights.logical_rows(), weights.width().n(),
        int(weight_plane), C.c_void_p(x.data_ptr()), features.logical_rows(),
        features.width().n(), int(feature_plane), k, C.c_void_p(y.data_ptr()), None))
    return y.cpu().numpy()


def compute_plane_products(weights: PackedBitPlanes, features: PackedBitPlanes,
                           ctx: Context | None = None) -> PlaneProductStack:
    """kernel.cpp:146-157 on the GPU (debug / property path; matmul_ap never forms it)."""
    ctx = ctx or default_context()
    if weights.logical_cols() != features.logical_cols():
        raise DimensionMismatch(f"operands disagree on K: {weights.logical_cols()} vs "
                                f"{features.logical_cols()}")
    nw, nx = weights.width().n(), features.width().n()
    stack = np.empty((nw, nx, weights.logical_rows(), features.logical_rows()), dtype=np.int32)
    _check(ctx.lib.apmm_compute_plane_products(
        ctx.h, _ptr(weights.words()), weights.logical_rows(), nw, _ptr(features.words()),
        features.logical_rows(), nx, weights.logical_cols(), _ptr(stack)))
    return PlaneProductStack(weights.width(), features.width(), weights.logical_cols(), stack)


def recover(stack: PlaneProductStack, ctx: Context | None = None) -> np.ndarray:
    """kernel.cpp:159-181 on the GPU: sum of 2^(i+j) Y^(i,j) in int64, checked narrowing."""
    ctx = ctx or default_context()
    p = stack.products()
    y = np.empty((stack.rows(), stack.cols()), dtype=np.int32)
    _check(ctx.lib.apmm_recover(ctx.h, _ptr(p), stack.weight_width().n(),
                                stack.feature_width().n(), stack.k_logical(), stack.rows(),
                                stack.cols(), _ptr(y)))
    return y


def matmul_ap_dequant(weights: PackedBitPlanes, w_scales, w_granularity: Granularity,
                      features: PackedBitPlanes, x_scales, x_granularity: Granularity,
                      ctx: Context | None = None) -> np.ndarray:
    """matmul_ap + the CLI dequant epilogue (apmm.cpp:329-340), fused on the GPU."""
    ctx = ctx or default_context()
    if weights.logical_cols() != features.logical_cols():
        raise DimensionMismatch(f"operands disagree on K: {weights.logical_cols()} vs "
                                f"{features.logical_cols()}")
    ws = np.ascontiguousarray(w_scales, dtype=np.float64)
    xs = np.ascontiguousarray(x_scales, dtype=np.float64)
    if ws.size != (weights.logical_rows() if w_granularity == Granularity.PerRow else 1) or \
            xs.size != (features.logical_rows() if x_granularity == Granularity.PerRow else 1):
        raise LengthMismatch("scale count does not match granularity")
    out = np.empty((weights.logical_rows(), features.logical_rows()), dtype=np.float32)
    _check(ctx.lib.apmm_matmul_ap_dequant(
        ctx.h, _ptr(weights.words()), weights.logical_rows(), weights.width().n(), _ptr(ws),
        int(w_granularity), _ptr(features.words()), features.logical_rows(),
        features.width().n(), _ptr(xs), int(x_granularity), weights.logical_cols(), _ptr(out)))
    return out


def kernel_fn(ctx: Context | None = None):
    """The verify.hpp:23-24 KernelFn seam: (W, X, TileConfig) -> AccumMatrix."""

    def fn(w: PackedBitPlanes, x: PackedBitPlanes, config: TileConfig = TileConfig()):
        return matmul_ap(w, x, config, ctx)

    return fn


# ---- device API (torch CUDA tensors, stream-ordered on torch's current stream) -------------
def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def cu_matmul_ap(w_planes, rows_w: int, n_w: int, x_planes, rows_x: int, n_x: int, k: int,
                 y, ctx: Context | None = None, stream=None) -> None:
    """apmm_cu_matmul_ap on device buffers (torch tensors); y: int32 [rows_w, rows_x]."""
    ctx = ctx or default_context(w_planes.device.index or 0)
    _check(ctx.lib.apmm_cu_matmul_ap(ctx.h, C.c_void_p(w_planes.data_ptr()), rows_w, n_w,
                                     C.c_void_p(x_planes.data_ptr()), rows_x, n_x, k,
                                     C.c_void_p(y.data_ptr()), _stream_ptr(stream)))


def cu_matmul_ap_dequant(w_planes, rows_w, n_w, w_scales, w_gran, x_planes, rows_x, n_x,
                         x_scales, x_gran, k, out, ctx: Context | None = None,
                         stream=None) -> None:
    ctx = ctx or default_context(w_planes.device.index or 0)
    _check(ctx.lib.apmm_cu_matmul_ap_dequant(
        ctx.h, C.c_void_p(w_planes.data_ptr()), rows_w, n_w, C.c_void_p(w_scales.data_ptr()),
        int(w_gran), C.c_void_p(x_planes.data_ptr()), rows_x, n_x,
        C.c_void_p(x_scales.data_ptr()), int(x_gran), k, C.c_void_p(out.data_ptr()),
        _stream_ptr(stream)))


def cu_quantize_matmul_ap_dequant(w_planes, rows_w, n_w, w_scales, w_gran, x_values, rows_x, k,
                                  n_x, x_gran, x_scales, out, ctx: Context | None = None,
                                  stream=None) -> None:
    """quantize(X) -> matmul_ap -> dequant in one call (apmm.cpp:275-340), the quantizer
    writing the GEMM operand directly; x_scales receives X's scales (torch CUDA tensors)."""
    ctx = ctx or default_context(w_planes.device.index or 0)
    _check(ctx.lib.apmm_cu_quantize_matmul_ap_dequant(
        ctx.h, C.c_void_p(w_planes.data_ptr()), rows_w, n_w, C.c_void_p(w_scales.data_ptr()),
        int(w_gran), C.c_void_p(x_values.data_ptr()), rows_x, k, n_x, int(x_gran),
        C.c_void_p(x_scales.data_ptr()), C.c_void_p(out.data_ptr()), _stream_ptr(stream)))


def cu_pack(codes, rows, cols, n, planes, ctx: Context | None = None, stream=None) -> None:
    ctx = ctx or default_context(codes.device.index or 0)
    _check(ctx.lib.apmm_cu_pack(ctx.h, C.c_void_p(codes.data_ptr()), rows, cols, n,
                                C.c_void_p(planes.data_ptr()), _stream_ptr(stream)))


def cu_unpack(planes, rows, cols, n, codes, ctx: Context | None = None, stream=None) -> None:
    ctx = ctx or default_context(planes.device.index or 0)
    _check(ctx.lib.apmm_cu_unpack(ctx.h, C.c_void_p(planes.data_ptr()), rows, cols, n,
                                  C.c_void_p(codes.data_ptr()), _stream_ptr(stream)))


def cu_quantize_pack(values, rows, cols, n, gran, planes, scales, codes=None,
                     ctx: Context | None = None, stream=None) -> None:
    ctx = ctx or default_context(values.device.index or 0)
    _check(ctx.lib.apmm_cu_quantize_pack(
        ctx.h, C.c_void_p(values.data_ptr()), rows, cols, n, int(gran),
        C.c_void_p(planes.data_ptr()), C.c_void_p(scales.data_ptr()),
        C.c_void_p(codes.data_ptr() if codes is not None else 0), _stream_ptr(stream)))
