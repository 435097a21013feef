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
class ParseError(Error): pass
class IoError(Error): pass
class CudaError(Error): pass
class NoDevice(Error): pass
class UnsupportedDevice(Error): pass


_STATUS_TO_ERROR = {
    1: EvenValue, 2: OutOfRange, 3: NonFinite, 4: LengthMismatch, 5: DimensionMismatch,
    6: IndexOutOfBounds, 7: Overflow, 8: OverflowBound, 9: InvalidArgument, 10: ParseError,
    11: IoError, 100: CudaError,
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
class Route(enum.IntEnum):
    """Kernel routes (apmm_cuda.h APMM_ROUTE_*): schedules only, every route returns the same
    bits. AUTO picks by shape; the others pin one kernel (tests)."""
    AUTO = 0
    SKINNY = 1
    MID_SPLITK = 2
    PAIR = 3
    PAIR_WPLANES = 4
    PAIR_SPLITK = 5
    SINGLE_SM = 6
    TENSOR_CORE = 7
    STREAM_TC = 8


OPT_ROUTE, OPT_EARLY_WEIGHT_READ, OPT_EARLY_FEATURE_READ = 1, 2, 3


class Context:
    """Owns an apmm_ctx (one device, one bound stream, reusable workspace)."""

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

    def set_route(self, route: "Route") -> None:
        _check(self.lib.apmm_ctx_set_option(self.h, OPT_ROUTE, int(route)))

    def route(self) -> "Route":
        v = C.c_int()
        _check(self.lib.apmm_ctx_get_option(self.h, OPT_ROUTE, C.byref(v)))
        return Route(v.value)

    def set_early_weight_read(self, on: bool) -> None:
        _check(self.lib.apmm_ctx_set_option(self.h, OPT_EARLY_WEIGHT_READ, int(bool(on))))

    def set_early_feature_read(self, on: bool) -> None:
        """APMM_OPT_EARLY_FEATURE_READ: only when features are never produced by an
        early-triggering kernel launched right before a call (apmm_cuda.h)."""
        _check(self.lib.apmm_ctx_set_option(self.h, OPT_EARLY_FEATURE_READ, int(bool(on))))

    def reserve(self, rows_w: int, rows_x: int, k: int, n_w: int = 8) -> None:
        """Pre-size the workspace for calls up to this shape (before CUDA-graph capture)."""
        _check(self.lib.apmm_ctx_reserve(self.h, int(rows_w), int(rows_x), int(k), int(n_w)))

    def set_stream(self, stream) -> None:
        """Bind to a torch.cuda.Stream (or raw handle); see apmm_ctx_set_stream."""
        handle = getattr(stream, "cuda_stream", stream)
        _check(self.lib.apmm_ctx_set_stream(self.h, C.c_void_p(handle)))

    def enable_timing(self, enable: bool = True) -> None:
        _check(self.lib.apmm_ctx_enable_timing(self.h, int(bool(enable))))

    def kernel_time(self, kernel: int = 0):
        """(total device ms, launches) of kernel class 0=GEMM / 1=expand since last call."""
        ms, n = C.c_double(), C.c_uint64()
        _check(self.lib.apmm_ctx_kernel_time(self.h, int(kernel), C.byref(ms), C.byref(n)))
        return ms.value, int(n.value)


_tls = threading.local()


def default_context(device: int = 0, stream: int | None = None) -> Context:
    """Per-thread context for (device, stream). A context binds to one stream (its workspace
    is shared by its calls), so the device wrappers key theirs by the stream they enqueue
    on; the host API (stream None) uses the context's private stream."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    key = (device, stream)
    if key not in ctxs:
        ctxs[key] = Context(device)
    return ctxs[key]


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
    y = np.empty((weights.logical_rows(), features.logical_rows()), dtype=np.int32)
    _check(ctx.lib.apmm_matmul_plane_pair(
        ctx.h, _ptr(weights.words()), weights.logical_rows(), weights.width().n(),
        int(weight_plane), _ptr(features.words()), features.logical_rows(),
        features.width().n(), int(feature_plane), weights.logical_cols(), _ptr(y)))
    return y


def dot_1bit_xor(a, b, k_logical: int, ctx: Context | None = None) -> int:
    """kernel.cpp:115-123 on the GPU: k - 2 popc(a ^ b); OutOfRange for k == 0,
    LengthMismatch unless both hold exactly ceil(k/32) words."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    out = C.c_int64()
    _check(ctx.lib.apmm_dot_1bit_xor(ctx.h, _ptr(a), a.size, _ptr(b), b.size, int(k_logical),
                                     C.byref(out)))
    return int(out.value)


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


def _dctx(ctx, t, stream):
    """The context for a device call: the given one, else the thread's context for
    (device of t, the stream the call enqueues on)."""
    if ctx is not None:
        return ctx
    return default_context(t.device.index or 0, _stream_ptr(stream).value or 0)


def cu_matmul_ap(w_planes, rows_w: int, n_w: int, x_planes, rows_x: int, n_x: int, k: int,
                 y, ctx: Context | None = None, stream=None) -> None:
    """apmm_cu_matmul_ap on device buffers (torch tensors); y: int32 [rows_w, rows_x]."""
    ctx = _dctx(ctx, w_planes, stream)
    _check(ctx.lib.apmm_cu_matmul_ap(ctx.h, C.c_void_p(w_planes.data_ptr()), rows_w, n_w,
                                     C.c_void_p(x_planes.data_ptr()), rows_x, n_x, k,
                                     C.c_void_p(y.data_ptr()), _stream_ptr(stream)))


def cu_matmul_ap_dequant(w_planes, rows_w, n_w, w_scales, w_gran, x_planes, rows_x, n_x,
                         x_scales, x_gran, k, out, ctx: Context | None = None,
                         stream=None) -> None:
    ctx = _dctx(ctx, w_planes, stream)
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
    ctx = _dctx(ctx, w_planes, stream)
    _check(ctx.lib.apmm_cu_quantize_matmul_ap_dequant(
        ctx.h, C.c_void_p(w_planes.data_ptr()), rows_w, n_w, C.c_void_p(w_scales.data_ptr()),
        int(w_gran), C.c_void_p(x_values.data_ptr()), rows_x, k, n_x, int(x_gran),
        C.c_void_p(x_scales.data_ptr()), C.c_void_p(out.data_ptr()), _stream_ptr(stream)))


def cu_pack(codes, rows, cols, n, planes, ctx: Context | None = None, stream=None) -> None:
    ctx = _dctx(ctx, codes, stream)
    _check(ctx.lib.apmm_cu_pack(ctx.h, C.c_void_p(codes.data_ptr()), rows, cols, n,
                                C.c_void_p(planes.data_ptr()), _stream_ptr(stream)))


def cu_unpack(planes, rows, cols, n, codes, ctx: Context | None = None, stream=None) -> None:
    ctx = _dctx(ctx, planes, stream)
    _check(ctx.lib.apmm_cu_unpack(ctx.h, C.c_void_p(planes.data_ptr()), rows, cols, n,
                                  C.c_void_p(codes.data_ptr()), _stream_ptr(stream)))


def cu_quantize_pack(values, rows, cols, n, gran, planes, scales, codes=None,
                     ctx: Context | None = None, stream=None) -> None:
    ctx = _dctx(ctx, values, stream)
    _check(ctx.lib.apmm_cu_quantize_pack(
        ctx.h, C.c_void_p(values.data_ptr()), rows, cols, n, int(gran),
        C.c_void_p(planes.data_ptr()), C.c_void_p(scales.data_ptr()),
        C.c_void_p(codes.data_ptr() if codes is not None else 0), _stream_ptr(stream)))


def cu_dot_1bit_xor(a, b, k_logical: int, out, ctx: Context | None = None, stream=None) -> None:
    """apmm_cu_dot_1bit_xor: out (int64 device tensor, 1 element) <- k - 2 popc(a ^ b)."""
    ctx = _dctx(ctx, a, stream)
    _check(ctx.lib.apmm_cu_dot_1bit_xor(ctx.h, C.c_void_p(a.data_ptr()), a.numel(),
                                        C.c_void_p(b.data_ptr()), b.numel(), int(k_logical),
                                        C.c_void_p(out.data_ptr()), _stream_ptr(stream)))


def cu_matmul_ap_requant(w_planes, rows_w, n_w, w_scales, w_gran, x_planes, rows_x, n_x, x_scales,
                         x_gran, k, n_next, next_gran, yf, next_planes=None, next_scales=None,
                         absmax=None, ctx: Context | None = None, stream=None) -> None:
    """matmul_ap -> dequant -> the next layer's quantize + pack (apmm_cu_matmul_ap_requant).
    With `absmax` (device f64, rows_x or 1) the call stops after the GEMM and leaves the local
    maxima there (N-sharded layers reduce them across ranks, then cu_requant_pack)."""
    ctx = _dctx(ctx, w_planes, stream)

    def p(t):
        return C.c_void_p(t.data_ptr() if t is not None else 0)
    _check(ctx.lib.apmm_cu_matmul_ap_requant(
        ctx.h, p(w_planes), rows_w, n_w, p(w_scales), int(w_gran), p(x_planes), rows_x, n_x,
        p(x_scales), int(x_gran), k, n_next, int(next_gran), p(yf), p(next_planes),
        p(next_scales), p(absmax), _stream_ptr(stream)))


def cu_requant_pack(yf, rows_w, rows_x, absmax, n_next, next_gran, next_planes, next_scales,
                    ctx: Context | None = None, stream=None) -> None:
    """apmm_cu_requant_pack: quantize + pack X' = yf^T with the given absmax."""
    ctx = _dctx(ctx, yf, stream)
    _check(ctx.lib.apmm_cu_requant_pack(
        ctx.h, C.c_void_p(yf.data_ptr()), rows_w, rows_x, C.c_void_p(absmax.data_ptr()), n_next,
        int(next_gran), C.c_void_p(next_planes.data_ptr()), C.c_void_p(next_scales.data_ptr()),
        _stream_ptr(stream)))


# ---- APMM v1 tensor files (tensor_file.hpp:12-64) -------------------------------------------
class TensorKind(enum.IntEnum):
    Float32 = 0
    QuantizedBipolar = 1


class _TensorInfo(C.Structure):
    _fields_ = [("kind", C.c_int), ("bit_width", C.c_int), ("granularity", C.c_int),
                ("rows", C.c_uint64), ("cols", C.c_uint64), ("scale_count", C.c_uint64),
                ("payload_offset", C.c_uint64), ("payload_words", C.c_uint64)]


@dataclass
class TensorFile:
    """tensor_file.hpp:41-64. Header validation and parsing run in the C library
    (apmm_tensor_parse, the reference's checks and messages); the arrays are views of the
    file bytes."""
    kind: TensorKind
    bit_width: int
    granularity: int  # 0 per-tensor, 1 per-row, 0xFF for float
    rows: int
    cols: int
    scales: np.ndarray
    float_data: np.ndarray
    packed: np.ndarray
    _bytes: bytes = b""

    def to_packed(self) -> PackedBitPlanes:
        if self.kind != TensorKind.QuantizedBipolar:
            raise ParseError("tensor file is not the quantized kind")
        return PackedBitPlanes(self.rows, self.cols, BitWidth(self.bit_width), self.packed)

    def to_real(self) -> np.ndarray:
        if self.kind != TensorKind.Float32:
            raise ParseError("tensor file is not the float32 kind")
        return self.float_data.astype(np.float64).reshape(self.rows, self.cols)

    def granularity_enum(self) -> Granularity:
        if self.granularity in (0, 1):
            return Granularity(self.granularity)
        raise ParseError("tensor file carries no quantization granularity")

    def cu_upload(self, ctx: Context | None = None, stream=None):
        """Device copies straight from the file bytes (apmm_cu_tensor_upload): quantized ->
        (planes int32 tensor, scales f64 tensor); float -> f64 values [rows, cols]."""
        import torch
        ctx = ctx or default_context(torch.cuda.current_device(), _stream_ptr(stream).value or 0)
        dev = torch.device("cuda", ctx.device)
        buf = np.frombuffer(self._bytes, dtype=np.uint8)
        if self.kind == TensorKind.QuantizedBipolar:
            planes = torch.empty(self.packed.size, dtype=torch.int32, device=dev)
            scales = torch.empty(self.scales.size, dtype=torch.float64, device=dev)
            _check(ctx.lib.apmm_cu_tensor_upload(ctx.h, _ptr(buf), buf.size,
                                                 C.c_void_p(planes.data_ptr()),
                                                 C.c_void_p(scales.data_ptr()), None,
                                                 _stream_ptr(stream)))
            return planes, scales
        values = torch.empty((self.rows, self.cols), dtype=torch.float64, device=dev)
        _check(ctx.lib.apmm_cu_tensor_upload(ctx.h, _ptr(buf), buf.size, None, None,
                                             C.c_void_p(values.data_ptr()), _stream_ptr(stream)))
        return values


def parse_tensor(data: bytes) -> TensorFile:
    """tensor_file.cpp:159-229 (validation in the C library)."""
    data = bytes(data)
    buf = np.frombuffer(data, dtype=np.uint8)
    info = _TensorInfo()
    _check(_lib.load().apmm_tensor_parse(_ptr(buf) if buf.size else None, buf.size,
                                         C.byref(info)))
    off = info.payload_offset
    if info.kind == 1:
        scales = np.frombuffer(data, dtype="<f8", count=info.scale_count, offset=16).copy()
        packed = np.frombuffer(data, dtype="<u4", count=info.payload_words, offset=off).copy()
        return TensorFile(TensorKind.QuantizedBipolar, info.bit_width, info.granularity,
                          info.rows, info.cols, scales, np.empty(0, np.float32), packed, data)
    floats = np.frombuffer(data, dtype="<f4", count=info.payload_words, offset=off).copy()
    return TensorFile(TensorKind.Float32, 0, 0xFF, info.rows, info.cols, np.empty(0),
                      floats, np.empty(0, np.uint32), data)


def read_tensor_file(path) -> TensorFile:
    """tensor_file.cpp:231- (IoError when unreadable)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot open {path} for reading") from e
    return parse_tensor(data)


def serialize_tensor(t: TensorFile) -> bytes:
    """tensor_file.cpp:135-157 for the quantized kind (apmm_tensor_serialize_quantized)."""
    if t.kind != TensorKind.QuantizedBipolar:
        raise InvalidArgument("only the quantized kind is serialized by this library")
    lib = _lib.load()
    sc = np.ascontiguousarray(t.scales, dtype=np.float64)
    pk = np.ascontiguousarray(t.packed, dtype=np.uint32)
    n = C.c_uint64()
    _check(lib.apmm_tensor_serialize_quantized(t.rows, t.cols, t.bit_width, t.granularity,
                                               _ptr(sc), _ptr(pk), None, 0, C.byref(n)))
    out = np.empty(n.value, dtype=np.uint8)
    _check(lib.apmm_tensor_serialize_quantized(t.rows, t.cols, t.bit_width, t.granularity,
                                               _ptr(sc), _ptr(pk), _ptr(out), out.size,
                                               C.byref(n)))
    return out.tobytes()


def load_tensor_file(path, ctx: Context | None = None):
    """apmm_tensor_file_load: read + validate + upload into fresh device tensors (synchronous).
    Returns (TensorKind, tensors...) like TensorFile.cu_upload."""
    import torch
    ctx = ctx or default_context(torch.cuda.current_device())
    t = read_tensor_file(path)
    dev = torch.device("cuda", ctx.device)
    if t.kind == TensorKind.QuantizedBipolar:
        planes = torch.empty(t.packed.size, dtype=torch.int32, device=dev)
        scales = torch.empty(t.scales.size, dtype=torch.float64, device=dev)
        _check(ctx.lib.apmm_tensor_file_load(ctx.h, str(path).encode(), None,
                                             C.c_void_p(planes.data_ptr()),
                                             C.c_void_p(scales.data_ptr()), None))
        return t, planes, scales
    values = torch.empty((t.rows, t.cols), dtype=torch.float64, device=dev)
    _check(ctx.lib.apmm_tensor_file_load(ctx.h, str(path).encode(), None, None, None,
                                         C.c_void_p(values.data_ptr())))
    return t, values
