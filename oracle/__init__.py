"""TEST INFRASTRUCTURE ONLY -- the parity oracle for the B200 bipolar-INT matmul.

Two checkers live here, both CPU-only:

* ``Oracle``  -- ctypes binding of ``apmm_oracle.c``, a plain-C restatement of the
  reference path (every C function cites the reference file:line it follows).
* ``Reference`` -- ctypes binding of ``_ref/libapmm_ref.so``: the UNMODIFIED reference
  library compiled from ``/root/reference/proj/src`` by ``oracle/Makefile`` plus the thin
  ``ref_shim.cpp``. Present when it was built in the container (it travels to the GPU
  box as a built file); ``Reference.available()`` says whether it loaded.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this package -- as the checker, never as the thing
measured or shipped. The product (``paper_2409_17870_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libapmm_ref.so")

PER_TENSOR, PER_ROW = 0, 1
STATUS = {
    0: "OK", 1: "EvenValue", 2: "OutOfRange", 3: "NonFinite", 4: "LengthMismatch",
    5: "DimensionMismatch", 6: "IndexOutOfBounds", 7: "Overflow", 8: "OverflowBound",
    9: "InvalidArgument", 10: "ParseError", 11: "IoError",
}


class OracleError(Exception):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {what}" if what else self.name)


def build(force: bool = False, with_ref: bool = True) -> None:
    """Compile liboracle.so (and _ref/ when /root/reference is present)."""
    targets = ["oracle"]
    if with_ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    if force or not os.path.exists(ORACLE_SO) or ("ref" in targets and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def words_per_row(cols: int) -> int:
    return (cols + 31) // 32


u64, i32, i64, vp = C.c_uint64, C.c_int, C.c_int64, C.c_void_p


class Oracle:
    """Plain-C restatement of the reference (oracle/apmm_oracle.c)."""

    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            if not os.path.exists(ORACLE_SO):
                build(with_ref=False)
            lib = C.CDLL(ORACLE_SO)
            sig = {
                "orc_rng_fill": (None, [vp, u64, vp]),
                "orc_rng_seed": (None, [vp, u64]),
                "orc_random_codes": (None, [vp, u64, u64, i32, vp]),
                "orc_quantize": (i32, [vp, u64, u64, i32, i32, vp, vp]),
                "orc_dequantize": (None, [vp, u64, u64, i32, i32, vp, vp]),
                "orc_pack": (None, [vp, u64, u64, i32, vp]),
                "orc_unpack": (None, [vp, u64, u64, i32, vp]),
                "orc_check_padding": (i32, [vp, u64, u64, i32]),
                "orc_dot_1bit_xor": (i32, [vp, u64, vp, u64, u64, vp]),
                "orc_plane_products": (i32, [vp, u64, i32, vp, u64, i32, u64, vp]),
                "orc_recover": (i32, [vp, i32, i32, u64, u64, vp]),
                "orc_overflow_bound": (i64, [i32, i32, u64]),
                "orc_matmul_ap": (i32, [vp, u64, i32, vp, u64, i32, u64, u64, u64, u64, vp]),
                "orc_matmul_ap_mt": (i32, [vp, u64, i32, vp, u64, i32, u64, i32, vp]),
                "orc_naive_matmul": (i32, [vp, u64, vp, u64, u64, vp]),
                "orc_decoded_matmul": (i32, [vp, u64, i32, vp, u64, i32, u64, vp]),
                "orc_dequant_epilogue": (None, [vp, u64, u64, vp, i32, vp, i32, vp]),
                "orc_decode": (i32, [C.c_uint, i32]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(lib, name)
                fn.restype, fn.argtypes = res, args
            Oracle._lib = lib
        self.lib = Oracle._lib

    @staticmethod
    def _check(st, what=""):
        if st != 0:
            raise OracleError(st, what)

    # --- Rng (include/apmm/rng.hpp) ---
    class Rng:
        def __init__(self, oracle: "Oracle", seed: int):
            self.o = oracle
            self.state = np.zeros(313 * 8, dtype=np.uint8)  # uint64 mt[312] + int idx
            oracle.lib.orc_rng_seed(_p(self.state), seed)

        def next_u64(self, count: int = 1) -> np.ndarray:
            out = np.empty(count, dtype=np.uint64)
            self.o.lib.orc_rng_fill(_p(self.state), count, _p(out))
            return out

        def below(self, n: int) -> int:
            return int(self.next_u64(1)[0] % np.uint64(n))

        def range(self, lo: int, hi: int) -> int:
            return lo + self.below(hi - lo + 1)

        def random_codes(self, rows: int, cols: int, n: int) -> np.ndarray:
            out = np.empty((rows, cols), dtype=np.uint8)
            self.o.lib.orc_random_codes(_p(self.state), rows, cols, n, _p(out))
            return out

    def rng(self, seed: int) -> "Oracle.Rng":
        return Oracle.Rng(self, seed)

    # --- hot-path functions ---
    def quantize(self, x: np.ndarray, n: int, gran: int):
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows, cols = x.shape
        codes = np.empty((rows, cols), dtype=np.uint8)
        scales = np.empty(rows if gran == PER_ROW else 1, dtype=np.float64)
        self._check(self.lib.orc_quantize(_p(x), rows, cols, n, gran, _p(codes), _p(scales)))
        return codes, scales

    def dequantize(self, codes, n, gran, scales):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        out = np.empty(codes.shape, dtype=np.float64)
        scales = np.ascontiguousarray(scales, dtype=np.float64)
        self.lib.orc_dequantize(_p(codes), codes.shape[0], codes.shape[1], n, gran,
                                _p(scales), _p(out))
        return out

    def pack(self, codes: np.ndarray, n: int) -> np.ndarray:
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        rows, cols = codes.shape
        out = np.empty(n * rows * words_per_row(cols), dtype=np.uint32)
        self.lib.orc_pack(_p(codes), rows, cols, n, _p(out))
        return out

    def unpack(self, planes: np.ndarray, rows: int, cols: int, n: int) -> np.ndarray:
        planes = np.ascontiguousarray(planes, dtype=np.uint32)
        out = np.empty((rows, cols), dtype=np.uint8)
        self.lib.orc_unpack(_p(planes), rows, cols, n, _p(out))
        return out

    def check_padding(self, planes, rows, cols, n) -> int:
        planes = np.ascontiguousarray(planes, dtype=np.uint32)
        return self.lib.orc_check_padding(_p(planes), rows, cols, n)

    def dot_1bit_xor(self, a, b, k) -> int:
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.zeros(1, dtype=np.int64)
        self._check(self.lib.orc_dot_1bit_xor(_p(a), a.size, _p(b), b.size, k, _p(out)))
        return int(out[0])

    def plane_products(self, w, rows_w, n_w, x, rows_x, n_x, k) -> np.ndarray:
        stack = np.empty((n_w, n_x, rows_w, rows_x), dtype=np.int32)
        self._check(self.lib.orc_plane_products(_p(w), rows_w, n_w, _p(x), rows_x, n_x, k,
                                                _p(stack)))
        return stack

    def recover(self, stack: np.ndarray) -> np.ndarray:
        stack = np.ascontiguousarray(stack, dtype=np.int32)
        n_w, n_x, m, n = stack.shape
        out = np.empty((m, n), dtype=np.int32)
        self._check(self.lib.orc_recover(_p(stack), n_w, n_x, m, n, _p(out)))
        return out

    def overflow_bound(self, n_w, n_x, k) -> int:
        return int(self.lib.orc_overflow_bound(n_w, n_x, k))

    def matmul_ap(self, w, rows_w, n_w, x, rows_x, n_x, k, tile=(64, 64, 512)) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.uint32)
        x = np.ascontiguousarray(x, dtype=np.uint32)
        y = np.empty((rows_w, rows_x), dtype=np.int32)
        self._check(self.lib.orc_matmul_ap(_p(w), rows_w, n_w, _p(x), rows_x, n_x, k,
                                           tile[0], tile[1], tile[2], _p(y)))
        return y

    def matmul_ap_mt(self, w, rows_w, n_w, x, rows_x, n_x, k, threads) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.uint32)
        x = np.ascontiguousarray(x, dtype=np.uint32)
        y = np.empty((rows_w, rows_x), dtype=np.int32)
        self._check(self.lib.orc_matmul_ap_mt(_p(w), rows_w, n_w, _p(x), rows_x, n_x, k,
                                              threads, _p(y)))
        return y

    def naive_matmul(self, a, b_kmajor) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.int32)
        b = np.ascontiguousarray(b_kmajor, dtype=np.int32)
        y = np.empty((a.shape[0], b.shape[0]), dtype=np.int32)
        self._check(self.lib.orc_naive_matmul(_p(a), a.shape[0], _p(b), b.shape[0], a.shape[1],
                                              _p(y)))
        return y

    def decoded_matmul(self, w_codes, n_w, x_codes, n_x) -> np.ndarray:
        w_codes = np.ascontiguousarray(w_codes, dtype=np.uint8)
        x_codes = np.ascontiguousarray(x_codes, dtype=np.uint8)
        y = np.empty((w_codes.shape[0], x_codes.shape[0]), dtype=np.int32)
        self._check(self.lib.orc_decoded_matmul(_p(w_codes), w_codes.shape[0], n_w,
                                                _p(x_codes), x_codes.shape[0], n_x,
                                                w_codes.shape[1], _p(y)))
        return y

    def decode(self, codes: np.ndarray, n: int) -> np.ndarray:
        return 2 * codes.astype(np.int32) - ((1 << n) - 1)

    def dequant_epilogue(self, y, w_scales, w_gran, x_scales, x_gran) -> np.ndarray:
        y = np.ascontiguousarray(y, dtype=np.int32)
        out = np.empty(y.shape, dtype=np.float32)
        ws = np.ascontiguousarray(w_scales, dtype=np.float64)
        xs = np.ascontiguousarray(x_scales, dtype=np.float64)
        self.lib.orc_dequant_epilogue(_p(y), y.shape[0], y.shape[1], _p(ws), w_gran, _p(xs),
                                      x_gran, _p(out))
        return out


class Reference:
    """The reference library itself (oracle/_ref/libapmm_ref.so), when built."""

    _lib = None

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self):
        if Reference._lib is None:
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
            lib = C.CDLL(REF_SO)
            sig = {
                "ref_rng_draws": (None, [u64, u64, vp]),
                "ref_quantize": (i32, [vp, u64, u64, i32, i32, vp, vp]),
                "ref_pack": (i32, [vp, u64, u64, i32, vp]),
                "ref_unpack": (i32, [vp, u64, u64, i32, vp]),
                "ref_matmul_ap": (i32, [vp, u64, i32, vp, u64, i32, u64, u64, u64, u64, vp]),
                "ref_decoded_matmul": (i32, [vp, u64, i32, vp, u64, i32, u64, vp]),
                "ref_plane_products": (i32, [vp, u64, i32, vp, u64, i32, u64, vp, vp]),
                "ref_dot_1bit_xor": (i32, [vp, u64, vp, u64, u64, vp]),
                "ref_job_prepare": (vp, [vp, u64, i32, vp, u64, i32, u64, i32]),
                "ref_job_run": (C.c_double, [vp]),
                "ref_job_result": (None, [vp, vp]),
                "ref_job_free": (None, [vp]),
                "ref_run_verify": (i32, [u64, i32, u64, u64, vp, i32]),
                "ref_serialize_quantized": (i32, [vp, u64, u64, i32, i32, vp, u64, vp]),
                "ref_serialize_float": (i32, [vp, u64, u64, vp, u64, vp]),
                "ref_parse_to_packed": (i32, [vp, u64, vp, vp]),
                "ref_last_error": (C.c_char_p, []),
            }
            for name, (res, args) in sig.items():
                fn = getattr(lib, name)
                fn.restype, fn.argtypes = res, args
            Reference._lib = lib
        self.lib = Reference._lib

    def _check(self, st):
        if st != 0:
            raise OracleError(st, self.lib.ref_last_error().decode())

    def rng_draws(self, seed, count):
        out = np.empty(count, dtype=np.uint64)
        self.lib.ref_rng_draws(seed, count, _p(out))
        return out

    def quantize(self, x, n, gran):
        x = np.ascontiguousarray(x, dtype=np.float64)
        rows, cols = x.shape
        codes = np.empty((rows, cols), dtype=np.uint8)
        scales = np.empty(rows if gran == PER_ROW else 1, dtype=np.float64)
        self._check(self.lib.ref_quantize(_p(x), rows, cols, n, gran, _p(codes), _p(scales)))
        return codes, scales

    def pack(self, codes, n):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        rows, cols = codes.shape
        out = np.empty(n * rows * words_per_row(cols), dtype=np.uint32)
        self._check(self.lib.ref_pack(_p(codes), rows, cols, n, _p(out)))
        return out

    def unpack(self, planes, rows, cols, n):
        planes = np.ascontiguousarray(planes, dtype=np.uint32)
        out = np.empty((rows, cols), dtype=np.uint8)
        self._check(self.lib.ref_unpack(_p(planes), rows, cols, n, _p(out)))
        return out

    def matmul_ap(self, w, rows_w, n_w, x, rows_x, n_x, k, tile=(64, 64, 512)):
        w = np.ascontiguousarray(w, dtype=np.uint32)
        x = np.ascontiguousarray(x, dtype=np.uint32)
        y = np.empty((rows_w, rows_x), dtype=np.int32)
        self._check(self.lib.ref_matmul_ap(_p(w), rows_w, n_w, _p(x), rows_x, n_x, k,
                                           tile[0], tile[1], tile[2], _p(y)))
        return y

    def decoded_matmul(self, w_codes, n_w, x_codes, n_x):
        w_codes = np.ascontiguousarray(w_codes, dtype=np.uint8)
        x_codes = np.ascontiguousarray(x_codes, dtype=np.uint8)
        y = np.empty((w_codes.shape[0], x_codes.shape[0]), dtype=np.int32)
        self._check(self.lib.ref_decoded_matmul(_p(w_codes), w_codes.shape[0], n_w, _p(x_codes),
                                                x_codes.shape[0], n_x, w_codes.shape[1], _p(y)))
        return y

    def plane_products(self, w, rows_w, n_w, x, rows_x, n_x, k):
        stack = np.empty((n_w, n_x, rows_w, rows_x), dtype=np.int32)
        y = np.empty((rows_w, rows_x), dtype=np.int32)
        self._check(self.lib.ref_plane_products(_p(w), rows_w, n_w, _p(x), rows_x, n_x, k,
                                                _p(stack), _p(y)))
        return stack, y

    def dot_1bit_xor(self, a, b, k):
        a = np.ascontiguousarray(a, dtype=np.uint32)
        b = np.ascontiguousarray(b, dtype=np.uint32)
        out = np.zeros(1, dtype=np.int64)
        self._check(self.lib.ref_dot_1bit_xor(_p(a), a.size, _p(b), b.size, k, _p(out)))
        return int(out[0])

    def serialize_quantized(self, x, n, gran) -> bytes:
        """quantize -> TensorFile::from_quantized -> serialize_tensor (the reference's bytes)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        ln = np.zeros(1, dtype=np.uint64)
        self._check(self.lib.ref_serialize_quantized(_p(x), x.shape[0], x.shape[1], n, gran,
                                                     None, 0, _p(ln)))
        out = np.empty(int(ln[0]), dtype=np.uint8)
        self._check(self.lib.ref_serialize_quantized(_p(x), x.shape[0], x.shape[1], n, gran,
                                                     _p(out), out.size, _p(ln)))
        return out.tobytes()

    def serialize_float(self, x) -> bytes:
        x = np.ascontiguousarray(x, dtype=np.float64)
        ln = np.zeros(1, dtype=np.uint64)
        self._check(self.lib.ref_serialize_float(_p(x), x.shape[0], x.shape[1], None, 0, _p(ln)))
        out = np.empty(int(ln[0]), dtype=np.uint8)
        self._check(self.lib.ref_serialize_float(_p(x), x.shape[0], x.shape[1], _p(out), out.size,
                                                 _p(ln)))
        return out.tobytes()

    def parse_to_packed(self, data: bytes, words: int, scales: int):
        buf = np.frombuffer(bytes(data), dtype=np.uint8)
        w = np.empty(words, dtype=np.uint32)
        s = np.empty(scales, dtype=np.float64)
        self._check(self.lib.ref_parse_to_packed(_p(buf), buf.size, _p(w), _p(s)))
        return w, s

    def run_verify(self, seed=1, cases=1000, max_dim=32, max_k=200):
        passed = np.zeros(16, dtype=np.int32)
        n = self.lib.ref_run_verify(seed, cases, max_dim, max_k, _p(passed), 16)
        if n < 0:
            raise OracleError(-n, self.lib.ref_last_error().decode())
        return [bool(v) for v in passed[:n]], self.lib.ref_last_error().decode()

    class Job:
        """Row-sliced multi-thread matmul_ap (prepared once, timed per run())."""

        def __init__(self, ref, w, rows_w, n_w, x, rows_x, n_x, k, threads):
            self.ref = ref
            self.w = np.ascontiguousarray(w, dtype=np.uint32)
            self.x = np.ascontiguousarray(x, dtype=np.uint32)
            self.rows_w, self.rows_x = rows_w, rows_x
            self.h = ref.lib.ref_job_prepare(_p(self.w), rows_w, n_w, _p(self.x), rows_x, n_x,
                                             k, threads)
            if not self.h:
                raise OracleError(9, ref.lib.ref_last_error().decode())

        def run(self) -> float:
            return float(self.ref.lib.ref_job_run(self.h))

        def result(self) -> np.ndarray:
            y = np.empty((self.rows_w, self.rows_x), dtype=np.int32)
            self.ref.lib.ref_job_result(self.h, _p(y))
            return y

        def __del__(self):
            if getattr(self, "h", None):
                self.ref.lib.ref_job_free(self.h)
                self.h = None

    def job(self, w, rows_w, n_w, x, rows_x, n_x, k, threads):
        return Reference.Job(self, w, rows_w, n_w, x, rows_x, n_x, k, threads)
