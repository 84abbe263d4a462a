"""Host-side mirror of the reference's FPx API over the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference C++
library (/root/reference/proj/include/fpx/), with device tensors instead of
host std::vectors:

    reference (namespace fpx)                 here
    --------------------------------------    -------------------------------
    FpxFormat / SplitScheme (format.hpp)      FpxFormat / SplitScheme
    Error / ErrorCode (error.hpp)             FpxError / ErrorCode
    quantize_matrix (codec.hpp:66)            quantize_matrix    -> K0 kernel
    dequantize_reference (codec.hpp:72)       dequantize         -> K3 kernel
    effective_scale (codec.hpp:76)            effective_scale
    pack / unpack (prepack.hpp:84-86)         pack / unpack      -> K1 kernel
    gemm_packed (gemm.hpp:27-28)              gemm_packed        -> K2 kernel
                                              fp6_linear (torch-layout alias)

Matrices follow the reference layouts: weights row-major [rows, cols];
activations B col-major K x N, which is a contiguous torch tensor of shape
[N, K]; the result C is fp32 col-major padded-rows x N, i.e. a torch tensor
of shape [N, rows_p].  torch supplies device memory and streams only; every
byte of compute runs in libfpx_b200.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field

import torch

from . import _lib

__all__ = [
    "ErrorCode", "FpxError", "FpxFormat", "SplitScheme", "QuantizedMatrix", "PackedWeights",
    "quantize_matrix", "pack", "unpack", "dequantize", "gemm_packed", "fp6_linear", "effective_scale",
    "linear_workspace", "default_split", "serialize_packed", "deserialize_packed", "write_pack_file",
    "read_pack_file", "linear", "quantize_pack",
]


class ErrorCode(enum.IntEnum):
    """error.hpp:10-24 (value = status - 1)."""
    InvalidFormat = 0
    InvalidCode = 1
    InvalidValue = 2
    ScaleOverflow = 3
    ShapeMismatch = 4
    RaggedInput = 5
    UnsupportedSplit = 6
    IndexOutOfRange = 7
    BadMagic = 8
    BadVersion = 9
    Truncated = 10
    Corrupt = 11
    IoFailure = 12


class FpxError(RuntimeError):
    """fpx::Error (error.hpp:30-44): code + message (+ optional byte offset)."""

    def __init__(self, status: int, message: str, offset: int | None = None):
        super().__init__(message)
        self.status = status
        self.code = ErrorCode(status - 1) if 1 <= status <= 13 else None
        self.offset = offset

    def formatted(self) -> str:
        return str(self)


def _check(status: int) -> None:
    if status != 0:
        L = _lib.load()
        off = int(L.fpx_last_error_offset())
        raise FpxError(status, L.fpx_last_error().decode(), off if off >= 0 else None)


@dataclass(frozen=True)
class FpxFormat:
    """format.hpp:16-45 -- sign + E + M bits, bias 2^(E-1)-1, no inf/nan."""
    exp_bits: int = 3
    man_bits: int = 2

    @property
    def total_bits(self) -> int:
        return 1 + self.exp_bits + self.man_bits

    @property
    def bias(self) -> int:
        return (1 << (self.exp_bits - 1)) - 1

    def max_representable(self) -> float:
        return float(_lib.load().fpx_max_representable(self.exp_bits, self.man_bits))

    def name(self) -> str:
        return f"e{self.exp_bits}m{self.man_bits}"

    @staticmethod
    def make(exp_bits: int, man_bits: int) -> "FpxFormat":
        _check(_lib.load().fpx_format_check(exp_bits, man_bits))
        return FpxFormat(exp_bits, man_bits)

    @staticmethod
    def parse(name: str) -> "FpxFormat | None":
        if len(name) != 4 or name[0] != "e" or name[2] != "m" or not name[1].isdigit() or not name[3].isdigit():
            return None
        try:
            return FpxFormat.make(int(name[1]), int(name[3]))
        except FpxError:
            return None

    e3m2 = None  # replaced below by constructors (FpxFormat.e3m2())


FpxFormat.e3m2 = staticmethod(lambda: FpxFormat(3, 2))  # type: ignore[assignment]
FpxFormat.e2m3 = staticmethod(lambda: FpxFormat(2, 3))  # type: ignore[attr-defined]
FpxFormat.e2m2 = staticmethod(lambda: FpxFormat(2, 2))  # type: ignore[attr-defined]
FpxFormat.e2m1 = staticmethod(lambda: FpxFormat(2, 1))  # type: ignore[attr-defined]


@dataclass(frozen=True)
class SplitScheme:
    """format.hpp:50-59 -- segment widths, most-significant first."""
    widths: tuple

    def total(self) -> int:
        return sum(self.widths)

    @staticmethod
    def for_format(fmt: FpxFormat) -> "SplitScheme":
        w = (C.c_int * 3)()
        n = _lib.load().fpx_split_for_format(fmt.exp_bits, fmt.man_bits, w)
        if n == 0:
            raise FpxError(1, f"error[invalid-format] no split for {fmt.name()}")
        return SplitScheme(tuple(w[i] for i in range(n)))

    @staticmethod
    def make(widths, fmt: FpxFormat) -> "SplitScheme":
        widths = tuple(int(x) for x in widths)
        if any(w not in (1, 2, 4) for w in widths):
            raise FpxError(7, "error[unsupported-split] segment widths must be 1, 2 or 4")
        if sum(widths) != fmt.total_bits:
            raise FpxError(7, f"error[unsupported-split] segment widths must sum to {fmt.total_bits} for {fmt.name()}")
        return SplitScheme(widths)


@dataclass
class QuantizedMatrix:
    """codec.hpp:37-51 on device: codes uint8 [rows, cols] (padded to 64), scales fp16 bits [rows]."""
    format: FpxFormat
    rows: int
    cols: int
    orig_rows: int
    orig_cols: int
    codes: torch.Tensor
    scales: torch.Tensor


@dataclass
class PackedWeights:
    """prepack.hpp:64-80 on device: one uint8 stream per segment + fp16-bit scales."""
    format: FpxFormat
    split: SplitScheme
    rows: int
    cols: int
    orig_rows: int
    orig_cols: int
    streams: list = field(default_factory=list)
    scales: torch.Tensor | None = None

    def tile_rows(self) -> int:
        return self.rows // 64

    def tile_cols(self) -> int:
        return self.cols // 64

    @staticmethod
    def tile_stream_bytes(w: int) -> int:
        return 512 * w

    @staticmethod
    def concat_rows(parts: list) -> "PackedWeights":
        """The inverse of shard(): several packed weights with the same format,
        split and padded K stacked along the output rows into ONE packed
        weight (a byte concatenation of every stream and of the scales, since
        tiles are stored in row-major tile order).  Linears that read the same
        activations -- gate and up of a LLaMA MLP, separate Q / K / V -- then
        run as one launch.  Part i's rows start at the sum of the previous
        parts' padded row counts; padding rows stay (code 0, zero output)."""
        if not parts:
            raise FpxError(3, "error[invalid-value] nothing to concatenate")
        p0 = parts[0]
        for p in parts[1:]:
            if (p.format.exp_bits, p.format.man_bits) != (p0.format.exp_bits, p0.format.man_bits) or \
                    p.split.widths != p0.split.widths or p.cols != p0.cols:
                raise FpxError(5, "error[shape-mismatch] concat_rows needs one format, split and padded K")
        streams = [torch.cat([p.streams[i].reshape(-1) for p in parts]) for i in range(len(p0.streams))]
        rows = sum(p.rows for p in parts)
        return PackedWeights(p0.format, p0.split, rows, p0.cols, rows, p0.orig_cols, streams,
                             torch.cat([p.scales for p in parts]))

    def shard(self, tr0: int, tr1: int) -> "PackedWeights":
        """Tile-rows [tr0, tr1) as zero-copy views (tiles are stored in
        row-major tile order, prepack.cpp:190-191, so a tile-row range is one
        contiguous byte range of every stream)."""
        gc = self.tile_cols()
        views = [s[tr0 * gc * 512 * w: tr1 * gc * 512 * w] for s, w in zip(self.streams, self.split.widths)]
        rows = (tr1 - tr0) * 64
        return PackedWeights(self.format, self.split, rows, self.cols, rows, self.orig_cols, views,
                             self.scales[tr0 * 64: tr1 * 64])


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _on(device: torch.device):
    """Make `device` current around a C-ABI call: the library queries the
    current device (sm_100 gate, SM count, per-device kernel attributes)."""
    return torch.cuda.device(device)


def pad64(n: int) -> int:
    return (n + 63) // 64 * 64


def effective_scale(row_scale: int, fmt: FpxFormat) -> int:
    """codec.cpp:195-199: fp16(scale * 2^(15 - bias))."""
    return int(_lib.load().fpx_effective_scale(row_scale, fmt.exp_bits, fmt.man_bits))


def quantize_matrix(m: torch.Tensor, fmt: FpxFormat) -> QuantizedMatrix:
    """codec.cpp:105-177: row-wise FPx quantisation on the GPU (bit-exact).

    m: CUDA tensor [rows, cols], fp32 (or fp16: converted exactly, codec.cpp:35-40).
    Raises FpxError(InvalidValue / ScaleOverflow / ShapeMismatch) like the reference."""
    L = _lib.load()
    if m.dim() != 2 or not m.is_cuda:
        raise FpxError(3, "error[invalid-value] quantize expects a row-major fp32 matrix")
    if m.dtype == torch.float32:
        dt = 0
    elif m.dtype == torch.float16:
        dt = 1
    else:
        raise FpxError(3, "error[invalid-value] quantize expects a row-major fp32 matrix")
    rows, cols = m.shape
    if rows == 0 or cols == 0:
        raise FpxError(5, "error[shape-mismatch] empty matrix")
    m = m.contiguous()
    rp, cp = pad64(rows), pad64(cols)
    codes = torch.empty((rp, cp), dtype=torch.uint8, device=m.device)
    scales = torch.empty((rp,), dtype=torch.int16, device=m.device)
    with _on(m.device):
        _check(L.fpx_quantize(m.data_ptr(), dt, rows, cols, fmt.exp_bits, fmt.man_bits, codes.data_ptr(),
                              scales.data_ptr(), None, _stream(m.device)))
    return QuantizedMatrix(fmt, rp, cp, rows, cols, codes, scales)


def pack(q: QuantizedMatrix, split: SplitScheme | None = None) -> PackedWeights:
    """prepack.cpp:153-209: ahead-of-time bit-level pre-pack (bit-exact bytes)."""
    L = _lib.load()
    split = split or SplitScheme.for_format(q.format)
    dev = q.codes.device
    streams = [torch.empty(L.fpx_stream_bytes(q.rows, q.cols, w), dtype=torch.uint8, device=dev)
               for w in split.widths]
    wid = (C.c_int * len(split.widths))(*split.widths)
    ptrs = (C.c_void_p * len(streams))(*[s.data_ptr() for s in streams])
    with _on(dev):
        _check(L.fpx_prepack(q.codes.data_ptr(), q.scales.data_ptr(), q.rows, q.cols, q.format.exp_bits,
                             q.format.man_bits, wid, len(split.widths), ptrs, _stream(dev)))
    return PackedWeights(q.format, split, q.rows, q.cols, q.orig_rows or q.rows, q.orig_cols or q.cols, streams,
                         q.scales.clone())


def quantize_pack(m: torch.Tensor, fmt: FpxFormat, split: SplitScheme | None = None) -> PackedWeights:
    """pack(quantize_matrix(m, fmt)) in one fused GPU pass (fpx_quantize_pack):
    bit-exact with the two-step path, without the code matrix in HBM."""
    L = _lib.load()
    if m.dim() != 2 or not m.is_cuda or m.dtype not in (torch.float32, torch.float16):
        raise FpxError(3, "error[invalid-value] quantize expects a row-major fp32 matrix")
    rows, cols = m.shape
    if rows == 0 or cols == 0:
        raise FpxError(5, "error[shape-mismatch] empty matrix")
    m = m.contiguous()
    split = split or SplitScheme.for_format(fmt)
    rp, cp = pad64(rows), pad64(cols)
    streams = [torch.empty(L.fpx_stream_bytes(rp, cp, w), dtype=torch.uint8, device=m.device) for w in split.widths]
    scales = torch.empty((rp,), dtype=torch.int16, device=m.device)
    wid = (C.c_int * len(split.widths))(*split.widths)
    ptrs = (C.c_void_p * len(streams))(*[s.data_ptr() for s in streams])
    with _on(m.device):
        _check(L.fpx_quantize_pack(m.data_ptr(), 0 if m.dtype == torch.float32 else 1, rows, cols, fmt.exp_bits,
                                   fmt.man_bits, wid, len(split.widths), ptrs, scales.data_ptr(), None,
                                   _stream(m.device)))
    return PackedWeights(fmt, split, rp, cp, rows, cols, streams, scales)


def unpack(p: PackedWeights) -> QuantizedMatrix:
    """prepack.cpp:211-260: exact inverse of pack."""
    L = _lib.load()
    dev = p.streams[0].device
    codes = torch.empty((p.rows, p.cols), dtype=torch.uint8, device=dev)
    wid = (C.c_int * len(p.split.widths))(*p.split.widths)
    ptrs = (C.c_void_p * len(p.streams))(*[s.data_ptr() for s in p.streams])
    with _on(dev):
        _check(L.fpx_unpack(ptrs, p.rows, p.cols, p.format.exp_bits, p.format.man_bits, wid, len(p.split.widths),
                            codes.data_ptr(), _stream(dev)))
    return QuantizedMatrix(p.format, p.rows, p.cols, p.orig_rows, p.orig_cols, codes, p.scales.clone())


def dequantize(p: PackedWeights) -> torch.Tensor:
    """fp16 W [rows_p, cols_p] from the packed streams; bit-exact with the
    reference's dequantize_reference (codec.cpp:179-193)."""
    L = _lib.load()
    dev = p.streams[0].device
    out = torch.empty((p.rows, p.cols), dtype=torch.float16, device=dev)
    wid = (C.c_int * len(p.split.widths))(*p.split.widths)
    ptrs = (C.c_void_p * len(p.streams))(*[s.data_ptr() for s in p.streams])
    with _on(dev):
        _check(L.fpx_dequantize(ptrs, len(p.streams), wid, p.scales.data_ptr(), p.rows, p.cols, p.format.exp_bits,
                                p.format.man_bits, out.data_ptr(), _stream(dev)))
    return out


_ws_lock = threading.Lock()
_ws: dict = {}


def linear_workspace(device: torch.device, nbytes: int) -> torch.Tensor | None:
    """Per (device, stream) zero-initialised workspace, grown on demand. Its
    split-K counter table self-cleans after every launch."""
    if nbytes == 0:
        return None
    key = (device.index if device.index is not None else torch.cuda.current_device(), _stream(device))
    with _ws_lock:
        buf = _ws.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            _ws[key] = buf
        return buf


def default_split(rows_p: int, cols_p: int, n: int) -> int:
    return int(_lib.load().fpx_linear_default_split(rows_p, cols_p, n))


def gemm_packed(p: PackedWeights, b: torch.Tensor, *, out: torch.Tensor | None = None, split_k: int = 0,
                ldc: int | None = None) -> torch.Tensor:
    """gemm.cpp:170-219: C = dequant(A) x B on the fused sm_100a kernel.

    b: fp16 activations, col-major K x N == contiguous torch [N, K] with
       K == p.cols or p.orig_cols (zero-extended, gemm.cpp:15-30).
    returns C fp32 col-major rows_p x N == torch [N, rows_p] (padded rows kept,
       like the reference).  `out` may be a preallocated [N, ldc] fp32 tensor.
    split_k: K chunks per 128-row tile (0 = default); results depend only on
       (inputs, split_k)."""
    L = _lib.load()
    if b.dtype != torch.float16 or b.dim() != 2:
        raise FpxError(5, "error[shape-mismatch] activations must be fp16 col-major")
    dev = p.streams[0].device
    if not b.is_cuda or b.device != dev:
        raise FpxError(3, f"error[invalid-value] activations must live on the weights' device {dev}")
    n, k_act = b.shape
    if k_act != p.cols and k_act != p.orig_cols:
        raise FpxError(5, f"error[shape-mismatch] weight cols {p.cols} (orig {p.orig_cols}) do not match "
                          f"activation rows {k_act}")
    b = b.contiguous()
    if out is None:
        ldc = ldc or p.rows
        out = torch.empty((n, ldc), dtype=torch.float32, device=dev)
    else:
        if out.dtype != torch.float32 or out.dim() != 2 or not out.is_contiguous() or out.device != dev:
            raise FpxError(5, "error[shape-mismatch] out must be a contiguous fp32 [N, ldc] tensor on the weights' "
                              "device")
        if ldc is not None and ldc != out.shape[1]:
            raise FpxError(5, f"error[shape-mismatch] ldc {ldc} != out.shape[1] {out.shape[1]}")
        ldc = out.shape[1]
        if out.shape[0] != n or ldc < p.rows:
            raise FpxError(5, f"error[shape-mismatch] out must be [{n}, >= {p.rows}], got {list(out.shape)}")
    if n == 0:
        return out
    sk = split_k if split_k > 0 else default_split(p.rows, p.cols, n)
    misaligned = b.data_ptr() % 16 != 0
    with _on(dev):
        need = int(L.fpx_linear_workspace_size(p.rows, p.cols, k_act + (1 if misaligned else 0), n, sk))
        ws = linear_workspace(dev, need)
        ptrs = (C.c_void_p * len(p.streams))(*[s.data_ptr() for s in p.streams])
        _check(L.fpx_linear(ptrs, len(p.streams), p.scales.data_ptr(), p.rows, p.cols, p.format.exp_bits,
                            p.format.man_bits, b.data_ptr(), k_act, n, out.data_ptr(), ldc, sk,
                            _ptr(ws), 0 if ws is None else ws.numel(), _stream(dev)))
    return out


# ------------------------------------------------------------ PackFile I/O
# io.hpp:30-37 (serialize_packed / deserialize_packed / write_pack_file /
# read_pack_file), the FPXPACK1 container of include/fpx_c.h.

def serialize_packed(p: PackedWeights) -> bytes:
    """io.hpp:30: PackedWeights -> FPXPACK1 bytes (little-endian, bit-exact)."""
    import numpy as np
    L = _lib.load()
    wid = (C.c_int * len(p.split.widths))(*p.split.widths)
    host = [s.detach().contiguous().cpu().numpy() for s in p.streams]
    scales = p.scales.detach().contiguous().cpu().numpy().view(np.uint16)
    n = int(L.fpx_packfile_bytes(p.rows, p.cols, wid, len(p.split.widths)))
    out = np.empty(n, dtype=np.uint8)
    ptrs = (C.c_void_p * len(host))(*[h.ctypes.data for h in host])
    _check(L.fpx_packfile_encode(p.format.exp_bits, p.format.man_bits, wid, len(p.split.widths), p.orig_rows,
                                 p.orig_cols, p.rows, p.cols, scales.ctypes.data, ptrs, out.ctypes.data, n))
    return out.tobytes()


def _from_header(h, scales: torch.Tensor, streams: list) -> PackedWeights:
    fmt = FpxFormat(h.exp_bits, h.man_bits)
    split = SplitScheme(tuple(h.widths[i] for i in range(h.nseg)))
    return PackedWeights(fmt, split, h.rows_p, h.cols_p, h.orig_rows, h.orig_cols, streams, scales)


def deserialize_packed(data: bytes, device: str | torch.device = "cpu") -> PackedWeights:
    """io.hpp:31: strict validation (FpxError BadMagic / BadVersion /
    Truncated / Corrupt with the byte offset), then the tensors on `device`."""
    import numpy as np
    L = _lib.load()
    buf = np.frombuffer(data, dtype=np.uint8)
    h = _lib.PackHeader()
    _check(L.fpx_packfile_parse(buf.ctypes.data if buf.size else None, buf.size, C.byref(h)))
    sc = torch.from_numpy(buf[h.scales_offset: h.scales_offset + 2 * h.rows_p].copy().view(np.int16))
    streams = [torch.from_numpy(buf[h.stream_offset[i]: h.stream_offset[i] + h.stream_bytes[i]].copy())
               for i in range(h.nseg)]
    return _from_header(h, sc.to(device), [t.to(device) for t in streams])


def write_pack_file(path: str, p: PackedWeights) -> None:
    """io.hpp:36."""
    data = serialize_packed(p)
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise FpxError(13, f"error[io-failure] cannot write {path}: {e}")


def read_pack_file(path: str, device: str | torch.device = "cuda") -> PackedWeights:
    """io.hpp:37.  On a CUDA device the payload goes straight from disk into
    device buffers (fpx_packfile_load: pinned staging, no pageable copy)."""
    L = _lib.load()
    dev = torch.device(device)
    h = _lib.PackHeader()
    if dev.type != "cuda":
        try:
            with open(path, "rb") as f:
                data = f.read()
        except OSError as e:
            raise FpxError(13, f"error[io-failure] cannot open {path}: {e}")
        return deserialize_packed(data, dev)
    _check(L.fpx_packfile_load(path.encode(), C.byref(h), None, None, None))  # validate, sizes
    scales = torch.empty(h.rows_p, dtype=torch.int16, device=dev)
    streams = [torch.empty(h.stream_bytes[i], dtype=torch.uint8, device=dev) for i in range(h.nseg)]
    ptrs = (C.c_void_p * h.nseg)(*[t.data_ptr() for t in streams])
    with _on(dev):
        _check(L.fpx_packfile_load(path.encode(), C.byref(h), scales.data_ptr(), ptrs, _stream(dev)))
    return _from_header(h, scales, streams)


ACTIVATIONS = {None: 0, "none": 0, "relu": 1, "silu": 2, "gelu_tanh": 3}


def linear(act: torch.Tensor, p: PackedWeights, *, bias: torch.Tensor | None = None, activation: str | None = None,
           residual: torch.Tensor | None = None, out_dtype: torch.dtype = torch.float16, split_k: int = 0,
           out: torch.Tensor | None = None) -> torch.Tensor:
    """The fused linear with the fp16-output epilogue (fpx_linear_ex):
    out[n, m] = activation(act[n] . W[m] + bias[m]) + residual[n, m], computed
    in fp32, stored as out_dtype (fp16 RNE or fp32).  act: [N, K] fp16 with K ==
    p.cols or p.orig_cols; bias: [p.rows] fp32 (or [orig_rows], zero-padded);
    residual: [N, p.rows] of out_dtype."""
    L = _lib.load()
    if act.dtype != torch.float16 or act.dim() != 2 or not act.is_cuda:
        raise FpxError(3, "error[invalid-value] activations must be a CUDA fp16 [N, K] tensor")
    if act.device != p.streams[0].device:
        raise FpxError(3, f"error[invalid-value] activations must live on the weights' device {p.streams[0].device}")
    if out_dtype not in (torch.float16, torch.float32):
        raise FpxError(3, "error[invalid-value] out_dtype must be float16 or float32")
    act = act.contiguous()
    n, k = act.shape
    dev = act.device
    if out is None:
        out = torch.empty((n, p.rows), dtype=out_dtype, device=dev)
    if out.dtype != out_dtype or out.shape != (n, p.rows) or not out.is_contiguous():
        raise FpxError(5, "error[shape-mismatch] out must be contiguous [N, rows_p] of out_dtype")
    if bias is not None:
        bias = bias.to(device=dev, dtype=torch.float32).contiguous()
        if bias.numel() < p.rows:
            bias = torch.nn.functional.pad(bias, (0, p.rows - bias.numel()))
    if residual is not None:
        if residual.dtype != out_dtype or residual.shape != (n, p.rows):
            raise FpxError(5, "error[shape-mismatch] residual must be [N, rows_p] of out_dtype")
        residual = residual.contiguous()
    if activation not in ACTIVATIONS:
        raise FpxError(3, f"error[invalid-value] activation must be one of {sorted(k for k in ACTIVATIONS if k)}")
    epi = _lib.Epilogue(1 if out_dtype == torch.float16 else 0, _ptr(bias), ACTIVATIONS[activation], _ptr(residual))
    with _on(dev):
        misaligned = act.data_ptr() % 16 != 0
        ws_bytes = int(L.fpx_linear_workspace_size(p.rows, p.cols, k + (1 if misaligned else 0), n, split_k))
        ws = linear_workspace(dev, ws_bytes)
        ptrs = (C.c_void_p * len(p.streams))(*[s.data_ptr() for s in p.streams])
        _check(L.fpx_linear_ex(ptrs, len(p.streams), p.scales.data_ptr(), p.rows, p.cols, p.format.exp_bits,
                               p.format.man_bits, act.data_ptr(), k, n, out.data_ptr(), p.rows, split_k, C.byref(epi),
                               _ptr(ws), ws_bytes, _stream(dev)))
    return out


def fp6_linear(act: torch.Tensor, packed: PackedWeights, **kw) -> torch.Tensor:
    """The paper's fp6_linear(A, packedW, scales) -> C with torch layouts:
    act [N, K] fp16 -> [N, rows_p] fp32 (scales live in `packed`)."""
    return gemm_packed(packed, act, **kw)
