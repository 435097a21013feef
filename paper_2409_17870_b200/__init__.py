"""B200-native (sm_100a) bipolar-INT arbitrary-precision matmul (arXiv 2409.17870).

The product is libapmm_b200.so (C ABI: include/apmm_cuda.h). This package holds its CUDA
sources (csrc/), the in-tree build (build.py), the Python mirror of the reference API
(apmm.py) and the N-sharded multi-GPU wrapper (shard.py).
"""
from .apmm import (  # noqa: F401
    BitWidth, CudaError, DimensionMismatch, Error, EvenValue, Granularity, IndexOutOfBounds,
    InvalidArgument, LengthMismatch, NoDevice, NonFinite, OutOfRange, Overflow, OverflowBound,
    PackedBitPlanes, QuantizedTensor, TileConfig, UnsupportedDevice, Context, default_context,
    decompose_and_pack, unpack, quantize, matmul_ap, matmul_ap_dequant, overflow_bound,
    kernel_fn, cu_matmul_ap, cu_matmul_ap_dequant, cu_pack, cu_unpack, cu_quantize_pack,
    PlaneProductStack, matmul_plane_pair, compute_plane_products, recover,
    cu_quantize_matmul_ap_dequant, Route, dot_1bit_xor, cu_dot_1bit_xor, cu_matmul_ap_requant,
    cu_requant_pack, ParseError, IoError, TensorKind, TensorFile, parse_tensor, read_tensor_file,
    serialize_tensor, load_tensor_file,
    version,
)
