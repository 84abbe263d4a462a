"""numpy front-end for the test oracles (TEST INFRASTRUCTURE ONLY).

Loads oracle/liboracle.so (the C restatement, fpx_oracle.c) and, when present,
oracle/_ref/libfpxref.so (the unmodified reference library + ref_shim.cpp).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfpxref.so")

_u8p = C.POINTER(C.c_uint8)
_u16p = C.POINTER(C.c_uint16)
_f32p = C.POINTER(C.c_float)


def build() -> None:
    """Compile liboracle.so (and _ref/ when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def pad64(n: int) -> int:
    return (n + 63) // 64 * 64


def split_for(e: int, m: int) -> list[int]:
    """format.cpp:59-69 preset split (restated)."""
    return {3: [2, 1], 4: [4], 5: [4, 1], 6: [2, 4], 7: [4, 2, 1], 8: [4, 4]}[1 + e + m]


class Oracle:
    """ctypes wrapper over liboracle.so (the C restatement)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_half_to_float.restype = C.c_float
        L.orc_half_to_float.argtypes = [C.c_uint16]
        L.orc_float_to_half.restype = C.c_uint16
        L.orc_float_to_half.argtypes = [C.c_float]
        L.orc_half_mul.restype = C.c_uint16
        L.orc_half_mul.argtypes = [C.c_uint16, C.c_uint16]
        L.orc_decode.restype = C.c_float
        L.orc_decode.argtypes = [C.c_uint32, C.c_int, C.c_int]
        L.orc_encode.restype = C.c_uint32
        L.orc_encode.argtypes = [C.c_double, C.c_int, C.c_int]
        L.orc_max_rep.restype = C.c_float
        L.orc_max_rep.argtypes = [C.c_int, C.c_int]
        L.orc_effective_scale.restype = C.c_uint16
        L.orc_effective_scale.argtypes = [C.c_uint16, C.c_int, C.c_int]
        L.orc_quantize.argtypes = [_f32p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, _u8p, _u16p,
                                   C.POINTER(C.c_int64)]
        L.orc_pack.argtypes = [_u8p, _u16p, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                               C.POINTER(C.c_int), C.c_int, C.POINTER(_u8p)]
        L.orc_unpack.argtypes = [C.POINTER(_u8p), C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                 C.POINTER(C.c_int), C.c_int, _u8p]
        L.orc_dequantize.argtypes = [_u8p, _u16p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, _u16p]
        L.orc_dequant_packed_e3m2.argtypes = [_u8p, _u8p, _u16p, C.c_uint32, C.c_uint32, _u16p]
        L.orc_gemm_reference.argtypes = [_u8p, _u16p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                         C.c_int, _u16p, C.c_uint32, C.c_uint32, _f32p]
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_fnv1a64.argtypes = [_u8p, C.c_size_t, C.c_uint64]
        L.orc_swar_thread_slice.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), _u16p, _u16p]

    # --- scalar helpers
    def half_to_float(self, h: int) -> float:
        return self.lib.orc_half_to_float(h)

    def float_to_half(self, f: float) -> int:
        return self.lib.orc_float_to_half(f)

    def half_mul(self, a: int, b: int) -> int:
        return self.lib.orc_half_mul(a, b)

    def decode(self, code: int, e: int, m: int) -> float:
        return self.lib.orc_decode(code, e, m)

    def encode(self, v: float, e: int, m: int) -> int:
        return self.lib.orc_encode(v, e, m)

    def effective_scale(self, s: int, e: int, m: int) -> int:
        return self.lib.orc_effective_scale(s, e, m)

    # --- matrix ops
    def quantize(self, w: np.ndarray, e: int, m: int):
        w = np.ascontiguousarray(w, dtype=np.float32)
        rows, cols = w.shape
        rp, cp = pad64(rows), pad64(cols)
        codes = np.zeros((rp, cp), np.uint8)
        scales = np.zeros(rp, np.uint16)
        fail = C.c_int64(-1)
        st = self.lib.orc_quantize(_p(w, _f32p), rows, cols, e, m, _p(codes, _u8p),
                                   _p(scales, _u16p), C.byref(fail))
        return st, codes, scales, fail.value

    def pack(self, codes: np.ndarray, scales: np.ndarray, e: int, m: int, widths=None):
        widths = widths or split_for(e, m)
        rp, cp = codes.shape
        streams = [np.zeros(rp * cp * w // 8, np.uint8) for w in widths]
        arr = (_u8p * len(widths))(*[_p(s, _u8p) for s in streams])
        wid = (C.c_int * len(widths))(*widths)
        st = self.lib.orc_pack(_p(np.ascontiguousarray(codes), _u8p), _p(np.ascontiguousarray(scales), _u16p),
                               rp, cp, e, m, wid, len(widths), arr)
        return st, streams

    def unpack(self, streams, rows_p: int, cols_p: int, e: int, m: int, widths=None):
        widths = widths or split_for(e, m)
        codes = np.zeros((rows_p, cols_p), np.uint8)
        arr = (_u8p * len(widths))(*[_p(s, _u8p) for s in streams])
        wid = (C.c_int * len(widths))(*widths)
        st = self.lib.orc_unpack(arr, rows_p, cols_p, e, m, wid, len(widths), _p(codes, _u8p))
        return st, codes

    def dequantize(self, codes: np.ndarray, scales: np.ndarray, e: int, m: int) -> np.ndarray:
        rp, cp = codes.shape
        out = np.zeros((rp, cp), np.uint16)
        self.lib.orc_dequantize(_p(np.ascontiguousarray(codes), _u8p), _p(np.ascontiguousarray(scales), _u16p),
                                rp, cp, e, m, _p(out, _u16p))
        return out

    def dequant_packed_e3m2(self, streams, scales: np.ndarray, rows_p: int, cols_p: int) -> np.ndarray:
        out = np.zeros((rows_p, cols_p), np.uint16)
        self.lib.orc_dequant_packed_e3m2(_p(streams[0], _u8p), _p(streams[1], _u8p),
                                         _p(np.ascontiguousarray(scales), _u16p), rows_p, cols_p, _p(out, _u16p))
        return out

    def gemm_reference(self, codes, scales, e, m, b_colmajor: np.ndarray, orig_cols=None):
        """b_colmajor: uint16 array shaped [n, b_rows] (col-major K x N)."""
        rp, cp = codes.shape
        b = np.ascontiguousarray(b_colmajor, dtype=np.uint16)
        n, b_rows = b.shape
        c = np.zeros((n, rp), np.float32)
        st = self.lib.orc_gemm_reference(_p(np.ascontiguousarray(codes), _u8p), _p(np.ascontiguousarray(scales), _u16p),
                                         rp, cp, orig_cols or cp, e, m, _p(b, _u16p), b_rows, n, _p(c, _f32p))
        return st, c

    def fnv1a64(self, *bufs) -> str:
        h = 0
        for b in bufs:
            b = np.ascontiguousarray(b).view(np.uint8).reshape(-1)
            h = self.lib.orc_fnv1a64(_p(b, _u8p), b.size, h)
        return "%016x" % h


class Reference:
    """ctypes wrapper over oracle/_ref/libfpxref.so (the unmodified reference)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_quantize.argtypes = [_f32p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, _u8p, _u16p]
        L.ref_pack.argtypes = [_u8p, _u16p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                               C.POINTER(_u8p)]
        L.ref_unpack.argtypes = [C.POINTER(_u8p), _u16p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, _u8p]
        L.ref_dequantize.argtypes = [_u8p, _u16p, C.c_uint32, C.c_uint32, C.c_int, C.c_int, _u16p]
        L.ref_effective_scale.restype = C.c_uint16
        L.ref_effective_scale.argtypes = [C.c_uint16, C.c_int, C.c_int]
        L.ref_float_to_half.restype = C.c_uint16
        L.ref_float_to_half.argtypes = [C.c_float]
        L.ref_half_to_float.restype = C.c_float
        L.ref_half_to_float.argtypes = [C.c_uint16]
        L.ref_half_mul.restype = C.c_uint16
        L.ref_half_mul.argtypes = [C.c_uint16, C.c_uint16]
        L.ref_decode.restype = C.c_float
        L.ref_decode.argtypes = [C.c_uint32, C.c_int, C.c_int]
        L.ref_encode.restype = C.c_uint32
        L.ref_encode.argtypes = [C.c_double, C.c_int, C.c_int]
        L.ref_prepare.restype = C.c_void_p
        L.ref_prepare.argtypes = [_u8p, _u16p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int]
        L.ref_release.argtypes = [C.c_void_p]
        L.ref_gemm_packed.argtypes = [C.c_void_p, _u16p, C.c_uint32, C.c_uint32, _f32p]
        L.ref_gemm_reference.argtypes = [C.c_void_p, _u16p, C.c_uint32, C.c_uint32, _f32p]
        L.ref_gemm_reference_codes.argtypes = [_u8p, _u16p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                               C.c_int, _u16p, C.c_uint32, C.c_uint32, _f32p]

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def quantize(self, w: np.ndarray, e: int, m: int):
        w = np.ascontiguousarray(w, dtype=np.float32)
        rows, cols = w.shape
        codes = np.zeros((pad64(rows), pad64(cols)), np.uint8)
        scales = np.zeros(pad64(rows), np.uint16)
        st = self.lib.ref_quantize(_p(w, _f32p), rows, cols, e, m, _p(codes, _u8p), _p(scales, _u16p))
        return st, codes, scales

    def pack(self, codes, scales, e, m, orig_rows=None, orig_cols=None):
        rp, cp = codes.shape
        streams = [np.zeros(rp * cp * w // 8, np.uint8) for w in split_for(e, m)]
        arr = (_u8p * len(streams))(*[_p(s, _u8p) for s in streams])
        st = self.lib.ref_pack(_p(np.ascontiguousarray(codes), _u8p), _p(np.ascontiguousarray(scales), _u16p),
                               rp, cp, orig_rows or rp, orig_cols or cp, e, m, arr)
        return st, streams

    def unpack(self, streams, scales, rows_p, cols_p, e, m):
        codes = np.zeros((rows_p, cols_p), np.uint8)
        arr = (_u8p * len(streams))(*[_p(s, _u8p) for s in streams])
        st = self.lib.ref_unpack(arr, _p(np.ascontiguousarray(scales), _u16p), rows_p, cols_p, e, m, _p(codes, _u8p))
        return st, codes

    def dequantize(self, codes, scales, e, m):
        rp, cp = codes.shape
        out = np.zeros((rp, cp), np.uint16)
        st = self.lib.ref_dequantize(_p(np.ascontiguousarray(codes), _u8p), _p(np.ascontiguousarray(scales), _u16p),
                                     rp, cp, e, m, _p(out, _u16p))
        return st, out

    def gemm_reference(self, codes, scales, e, m, b_colmajor: np.ndarray, orig_cols=None, orig_rows=None):
        """gemm.cpp:221-252 on (codes, scales) directly; b_colmajor uint16 [n, b_rows].
        Returns C as float32 [n, rows_p] (col-major rows_p x n)."""
        rp, cp = codes.shape
        b = np.ascontiguousarray(b_colmajor, dtype=np.uint16)
        n, b_rows = b.shape
        c = np.zeros((n, rp), np.float32)
        st = self.lib.ref_gemm_reference_codes(_p(np.ascontiguousarray(codes), _u8p),
                                               _p(np.ascontiguousarray(scales), _u16p), rp, cp, orig_rows or rp,
                                               orig_cols or cp, e, m, _p(b, _u16p), b_rows, n, _p(c, _f32p))
        if st:
            raise RuntimeError(self.last_error())
        return c

    def prepare(self, codes, scales, e, m, orig_rows=None, orig_cols=None):
        rp, cp = codes.shape
        h = self.lib.ref_prepare(_p(np.ascontiguousarray(codes), _u8p), _p(np.ascontiguousarray(scales), _u16p),
                                 rp, cp, orig_rows or rp, orig_cols or cp, e, m)
        if not h:
            raise RuntimeError(self.last_error())
        return RefHandle(self, h, rp)


class RefHandle:
    def __init__(self, ref: Reference, h, rows_p: int):
        self.ref, self.h, self.rows_p = ref, h, rows_p

    def _gemm(self, fn, b_colmajor: np.ndarray):
        b = np.ascontiguousarray(b_colmajor, dtype=np.uint16)
        n, b_rows = b.shape
        c = np.zeros((n, self.rows_p), np.float32)
        st = fn(self.h, _p(b, _u16p), b_rows, n, _p(c, _f32p))
        if st:
            raise RuntimeError(self.ref.last_error())
        return c

    def gemm_packed(self, b_colmajor):
        return self._gemm(self.ref.lib.ref_gemm_packed, b_colmajor)

    def gemm_reference(self, b_colmajor):
        return self._gemm(self.ref.lib.ref_gemm_reference, b_colmajor)

    def __del__(self):
        try:
            self.ref.lib.ref_release(self.h)
        except Exception:
            pass
