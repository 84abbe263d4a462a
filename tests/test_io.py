"""PackFile / MatrixFile containers (io.hpp:13-41, SPEC.md model-io) and the
`fpx` CLI on CPU: byte layout, strict validation with byte offsets, round
trips, the compression-ratio acceptance criterion.  No GPU needed (the
containers are host code); tests/test_gpu_parity.py drives the CLI's GPU
subcommands."""
import os
import struct
import subprocess

import numpy as np
import pytest
import torch

import paper_2401_14112_b200 as fpx
from paper_2401_14112_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2401_14112_b200", "build", "fpx")


def random_packed(rows=100, cols=150, e=3, m=2, seed=0):
    """A host PackedWeights with random stream bytes (containers do not
    interpret the payload)."""
    rng = np.random.default_rng(seed)
    fmt = fpx.FpxFormat(e, m)
    sp = fpx.SplitScheme.for_format(fmt)
    rp, cp = fpx.fpx.pad64(rows), fpx.fpx.pad64(cols)
    L = _lib.load()
    streams = [torch.from_numpy(rng.integers(0, 256, L.fpx_stream_bytes(rp, cp, w), dtype=np.uint8)) for w in sp.widths]
    scales = torch.from_numpy(rng.integers(1, 0x4000, rp).astype(np.int16))
    return fpx.PackedWeights(fmt, sp, rp, cp, rows, cols, streams, scales)


def parse_spec(b: bytes):
    """Independent reader written from the SPEC text alone."""
    assert b[:8] == b"FPXPACK1"
    ver, e, m, ns = struct.unpack_from("<HBBB", b, 8)
    widths = list(b[13:13 + ns])
    off = 13 + ns
    orig_r, orig_c, rp, cp, tm, tk = struct.unpack_from("<6I", b, off)
    off += 24
    gran = b[off]
    off += 1
    scales = np.frombuffer(b, dtype="<u2", count=rp, offset=off)
    off += 2 * rp
    streams = []
    for _ in range(ns):
        (ln,) = struct.unpack_from("<Q", b, off)
        off += 8
        streams.append(np.frombuffer(b, dtype=np.uint8, count=ln, offset=off))
        off += ln
    assert off == len(b)
    return dict(ver=ver, e=e, m=m, widths=widths, dims=(orig_r, orig_c, rp, cp, tm, tk), gran=gran, scales=scales,
                streams=streams)


@pytest.mark.parametrize("e,m", [(3, 2), (2, 3), (2, 2)])
def test_packfile_layout_and_round_trip(e, m):
    p = random_packed(100, 150, e, m, seed=e)
    b = fpx.serialize_packed(p)
    d = parse_spec(b)
    assert (d["ver"], d["e"], d["m"], d["gran"]) == (1, e, m, 0)
    assert d["widths"] == list(p.split.widths)
    assert d["dims"] == (100, 150, 128, 192, 64, 64)
    assert (d["scales"] == p.scales.numpy().view(np.uint16)).all()
    for s, t in zip(d["streams"], p.streams):
        assert (s == t.numpy()).all()
    q = fpx.deserialize_packed(b)
    assert (q.rows, q.cols, q.orig_rows, q.orig_cols, q.format, q.split) == (p.rows, p.cols, p.orig_rows,
                                                                               p.orig_cols, p.format, p.split)
    assert fpx.serialize_packed(q) == b  # bit-exact round trip


def test_packfile_file_round_trip(tmp_path):
    p = random_packed(64, 64)
    path = str(tmp_path / "w.fpxpack")
    fpx.write_pack_file(path, p)
    q = fpx.read_pack_file(path, device="cpu")
    assert fpx.serialize_packed(q) == open(path, "rb").read()


def _err(b: bytes):
    with pytest.raises(fpx.FpxError) as ei:
        fpx.deserialize_packed(b)
    return ei.value


def test_packfile_strict_validation():
    b = fpx.serialize_packed(random_packed(64, 128))
    e = _err(b"NOTAPACK" + b[8:])
    assert e.code == fpx.ErrorCode.BadMagic and e.offset == 0
    e = _err(b[:8] + struct.pack("<H", 2) + b[10:])
    assert e.code == fpx.ErrorCode.BadVersion and e.offset == 8
    for cut in (3, 9, 14, 30, 40, 50, len(b) - 1):
        e = _err(b[:cut])
        assert e.code == fpx.ErrorCode.Truncated and e.offset is not None and e.offset <= cut, (cut, e)
    e = _err(b + b"\0")
    assert e.code == fpx.ErrorCode.Corrupt and e.offset == len(b)
    # a stream length off the size law
    d = bytearray(b)
    off = 13 + 2 + 24 + 1 + 2 * 64
    struct.pack_into("<Q", d, off, 7)
    e = _err(bytes(d))
    assert e.code == fpx.ErrorCode.Corrupt and e.offset == off
    # inconsistent dimensions (padded != pad64(orig))
    d = bytearray(b)
    struct.pack_into("<I", d, 15 + 8, 192)
    assert _err(bytes(d)).code == fpx.ErrorCode.Corrupt
    # widths that do not split the format
    d = bytearray(b)
    d[13] = 1
    assert _err(bytes(d)).code == fpx.ErrorCode.UnsupportedSplit
    # tile shape
    d = bytearray(b)
    struct.pack_into("<I", d, 15 + 16, 32)
    assert _err(bytes(d)).code == fpx.ErrorCode.Corrupt


def test_compression_ratio_acceptance_4():
    """SPEC acceptance 4: 4096x4096 e3m2 -- streams / fp16 payload = 0.375
    exactly, whole PackFile / fp16 payload <= 0.40."""
    L = _lib.load()
    w = (__import__("ctypes").c_int * 2)(2, 4)
    fp16 = 4096 * 4096 * 2
    streams = L.fpx_stream_bytes(4096, 4096, 2) + L.fpx_stream_bytes(4096, 4096, 4)
    assert streams / fp16 == 0.375
    assert L.fpx_packfile_bytes(4096, 4096, w, 2) / fp16 <= 0.40


@pytest.mark.skipif(not os.path.exists(CLI), reason="CLI not built")
def test_cli_inspect_and_errors(tmp_path):
    p = random_packed(100, 150)
    path = str(tmp_path / "w.fpxpack")
    fpx.write_pack_file(path, p)
    r = subprocess.run([CLI, "inspect", "--input", path, "--tile", "1,2", "--thread", "5"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    assert "format e3m2  split 2 4  orig 100x150  padded 128x192" in r.stdout
    # the 2-bit segment's first word of thread 5 in tile (1,2): byte (j*32+t)*4 of the tile's 1 KB block
    tile = 1 * 3 + 2
    blk = p.streams[0].numpy()[tile * 1024: tile * 1024 + 1024]
    word = int.from_bytes(blk[5 * 4: 5 * 4 + 4].tobytes(), "little")
    assert f"{word:08x}" in r.stdout
    open(path, "r+b").truncate(200)
    r = subprocess.run([CLI, "inspect", "--input", path], capture_output=True, text=True)
    assert r.returncode == 3 and "error[truncated]" in r.stderr and "(at byte" in r.stderr
    assert subprocess.run([CLI, "bogus"], capture_output=True).returncode == 2
