"""ctypes binding of libfpx_b200.so (the C-ABI declared in include/fpx_c.h).

The shared library is built in-tree by `make -C paper_2401_14112_b200` (see
__graft_entry__.build()).  There is no fallback: if the library is missing
or fails to load, importing the compute API raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfpx_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "fpx_c.h")

_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)
_f32p = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_intp = C.POINTER(C.c_int)

_lib = None


class Epilogue(C.Structure):
    """fpx_epilogue (include/fpx_c.h)."""
    _fields_ = [("out_dtype", C.c_int), ("bias", C.c_void_p), ("activation", C.c_int), ("residual", C.c_void_p)]


class PackHeader(C.Structure):
    """fpx_pack_header (include/fpx_c.h)."""
    _fields_ = [("exp_bits", C.c_int), ("man_bits", C.c_int), ("nseg", C.c_int), ("widths", C.c_int * 3),
                ("orig_rows", C.c_uint32), ("orig_cols", C.c_uint32), ("rows_p", C.c_uint32), ("cols_p", C.c_uint32),
                ("scales_offset", C.c_uint64), ("stream_offset", C.c_uint64 * 3), ("stream_bytes", C.c_uint64 * 3),
                ("file_bytes", C.c_uint64)]


def header_symbols() -> list[str]:
    """Every function the public header declares (parsed from include/fpx_c.h)."""
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fpx_[a-z0-9_]+)\s*\(", text)))


def load(path: str | None = None) -> C.CDLL:
    """Load the in-tree library (FPX_B200_LIB may name an alternate in-tree
    build, e.g. a tuning variant from `make VARIANT=_x EXTRA=-D...`)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("FPX_B200_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run `make -C {HERE}` (or __graft_entry__.build())")
    L = C.CDLL(path)
    sig = {
        "fpx_last_error": (C.c_char_p, []),
        "fpx_status_name": (C.c_char_p, [C.c_int]),
        "fpx_version": (C.c_int, []),
        "fpx_format_check": (C.c_int, [C.c_int, C.c_int]),
        "fpx_split_for_format": (C.c_int, [C.c_int, C.c_int, _intp]),
        "fpx_max_representable": (C.c_float, [C.c_int, C.c_int]),
        "fpx_effective_scale": (C.c_uint16, [C.c_uint16, C.c_int, C.c_int]),
        "fpx_pad64": (C.c_uint32, [C.c_uint32]),
        "fpx_stream_bytes": (C.c_size_t, [C.c_uint32, C.c_uint32, C.c_int]),
        "fpx_quantize": (C.c_int, [C.c_void_p, C.c_int, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
        "fpx_linear_sharded_workspace_size": (C.c_size_t, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                                        C.c_int]),
        "fpx_linear_sharded": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int,
                                         C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_int,
                                         C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
        "fpx_quantize_pack": (C.c_int, [C.c_void_p, C.c_int, C.c_uint32, C.c_uint32, C.c_int, C.c_int, _intp, C.c_int,
                                        C.POINTER(C.c_void_p), C.c_void_p, C.c_void_p, C.c_void_p]),
        "fpx_prepack": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, _intp, C.c_int,
                                  C.POINTER(C.c_void_p), C.c_void_p]),
        "fpx_unpack": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.c_uint32, C.c_int, C.c_int, _intp, C.c_int,
                                 C.c_void_p, C.c_void_p]),
        "fpx_dequantize": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, _intp, C.c_void_p, C.c_uint32, C.c_uint32,
                                     C.c_int, C.c_int, C.c_void_p, C.c_void_p]),
        "fpx_linear_default_split": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32]),
        "fpx_linear_workspace_reset": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p]),
        "fpx_decode_scalar": (C.c_int, [C.c_uint32, C.c_int, C.c_int, _f32p]),
        "fpx_encode_scalar": (C.c_int, [C.c_double, C.c_int, C.c_int, _u32p]),
        "fpx_dequantize_codes": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                           C.c_void_p, C.c_void_p, C.c_void_p]),
        "fpx_linear_workspace_size": (C.c_size_t, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int]),
        "fpx_linear": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int,
                                 C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_int,
                                 C.c_void_p, C.c_size_t, C.c_void_p]),
        "fpx_last_error_offset": (C.c_int64, []),
        "fpx_linear_ex": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int,
                                    C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32, C.c_int,
                                    C.POINTER(Epilogue), C.c_void_p, C.c_size_t, C.c_void_p]),
        "fpx_packfile_bytes": (C.c_size_t, [C.c_uint32, C.c_uint32, _intp, C.c_int]),
        "fpx_packfile_encode": (C.c_int, [C.c_int, C.c_int, _intp, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p, C.c_size_t]),
        "fpx_packfile_parse": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(PackHeader)]),
        "fpx_packfile_load": (C.c_int, [C.c_char_p, C.POINTER(PackHeader), C.c_void_p, C.POINTER(C.c_void_p),
                                        C.c_void_p]),
        "fpx_debug_trace": (C.c_int, [C.c_void_p, C.c_size_t]),
        "fpx_debug_progress": (C.c_void_p, []),
        "fpx_shard_rows": (None, [C.c_uint32, C.c_int, C.c_int, _u32p, _u32p]),
        "fpx_gather_permute": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_uint32, C.c_uint32,
                                         C.c_void_p, C.c_uint32, C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
