"""paper_2401_14112_b200 -- B200-native (sm_100a) TC-FPx W6A16 linear layer.

A from-scratch re-design of the FP6-LLM (arXiv 2401.14112) weight path for
Blackwell: GPU quantize, bit-exact pre-pack, and a fused de-quantise +
tcgen05 GEMM behind the reference's API (see fpx.py) and a C-ABI
(include/fpx_c.h, libfpx_b200.so).
"""
from . import _lib  # noqa: F401
from .fpx import (  # noqa: F401
    ErrorCode, FpxError, FpxFormat, PackedWeights, QuantizedMatrix, SplitScheme, default_split, dequantize,
    deserialize_packed, effective_scale, fp6_linear, gemm_packed, linear, pack, quantize_pack, quantize_matrix, read_pack_file,
    serialize_packed, unpack, write_pack_file,
)
from . import shard  # noqa: F401,E402

__version__ = "0.1.0"
