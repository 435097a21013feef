"""ctypes loader for libapmm_b200.so (the C ABI of include/apmm_cuda.h).

Fails loudly: if the in-tree library is missing or does not load, every call raises --
there is no CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# APMM_LIB (dev only) points the loader at another build of the same ABI, e.g. to A/B a change
LIB_PATH = os.environ.get("APMM_LIB") or os.path.join(PKG, "libapmm_b200.so")

u64, i32, i64, vp = C.c_uint64, C.c_int, C.c_int64, C.c_void_p

_SIGNATURES = {
    "apmm_ctx_create": (i32, [C.POINTER(vp), i32]),
    "apmm_ctx_destroy": (i32, [vp]),
    "apmm_ctx_set_stream": (i32, [vp, vp]),
    "apmm_last_error": (C.c_char_p, []),
    "apmm_status_name": (C.c_char_p, [i32]),
    "apmm_version": (C.c_char_p, []),
    "apmm_ctx_launch_count": (u64, [vp]),
    "apmm_ctx_enable_timing": (i32, [vp, i32]),
    "apmm_ctx_kernel_time": (i32, [vp, i32, C.POINTER(C.c_double), C.POINTER(u64)]),
    "apmm_ctx_reserve": (i32, [vp, u64, u64, u64, i32]),
    "apmm_ctx_set_option": (i32, [vp, i32, i32]),
    "apmm_ctx_get_option": (i32, [vp, i32, C.POINTER(i32)]),
    "apmm_overflow_bound": (i32, [i32, i32, u64, C.POINTER(i64)]),
    "apmm_packed_words": (u64, [i32, u64, u64]),
    "apmm_cu_pack": (i32, [vp, vp, u64, u64, i32, vp, vp]),
    "apmm_cu_unpack": (i32, [vp, vp, u64, u64, i32, vp, vp]),
    "apmm_cu_quantize_pack": (i32, [vp, vp, u64, u64, i32, i32, vp, vp, vp, vp]),
    "apmm_cu_matmul_ap": (i32, [vp, vp, u64, i32, vp, u64, i32, u64, vp, vp]),
    "apmm_cu_matmul_ap_dequant": (i32, [vp, vp, u64, i32, vp, i32, vp, u64, i32, vp, i32, u64,
                                        vp, vp]),
    "apmm_cu_quantize_matmul_ap_dequant": (i32, [vp, vp, u64, i32, vp, i32, vp, u64, u64, i32, i32,
                                                 vp, vp, vp]),
    "apmm_cu_matmul_plane_pair": (i32, [vp, vp, u64, i32, i32, vp, u64, i32, i32, u64, vp, vp]),
    "apmm_cu_compute_plane_products": (i32, [vp, vp, u64, i32, vp, u64, i32, u64, vp, vp]),
    "apmm_cu_recover": (i32, [vp, vp, i32, i32, u64, u64, u64, vp, vp]),
    "apmm_cu_dot_1bit_xor": (i32, [vp, vp, u64, vp, u64, u64, vp, vp]),
    "apmm_cu_matmul_ap_requant": (i32, [vp, vp, u64, i32, vp, i32, vp, u64, i32, vp, i32, u64, i32,
                                        i32, vp, vp, vp, vp, vp]),
    "apmm_cu_requant_pack": (i32, [vp, vp, u64, u64, vp, i32, i32, vp, vp, vp]),
    "apmm_tensor_parse": (i32, [vp, u64, vp]),
    "apmm_cu_tensor_upload": (i32, [vp, vp, u64, vp, vp, vp, vp]),
    "apmm_tensor_file_load": (i32, [vp, C.c_char_p, vp, vp, vp, vp]),
    "apmm_tensor_serialize_quantized": (i32, [u64, u64, i32, i32, vp, vp, vp, u64,
                                              C.POINTER(u64)]),
    "apmm_dot_1bit_xor": (i32, [vp, vp, u64, vp, u64, u64, vp]),
    "apmm_matmul_plane_pair": (i32, [vp, vp, u64, i32, i32, vp, u64, i32, i32, u64, vp]),
    "apmm_compute_plane_products": (i32, [vp, vp, u64, i32, vp, u64, i32, u64, vp]),
    "apmm_recover": (i32, [vp, vp, i32, i32, u64, u64, u64, vp]),
    "apmm_decompose_and_pack": (i32, [vp, vp, u64, u64, i32, vp]),
    "apmm_unpack": (i32, [vp, vp, u64, u64, i32, vp]),
    "apmm_quantize_pack": (i32, [vp, vp, u64, u64, i32, i32, vp, vp, vp]),
    "apmm_matmul_ap": (i32, [vp, vp, u64, i32, vp, u64, i32, u64, vp]),
    "apmm_matmul_ap_dequant": (i32, [vp, vp, u64, i32, vp, i32, vp, u64, i32, vp, i32, u64, vp]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if absent and nvcc is available) the in-tree library."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from . import build as _build
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libapmm_b200.so not found at {LIB_PATH}; run "
                           f"`python -m paper_2409_17870_b200.build`")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib
