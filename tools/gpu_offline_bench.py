"""Ahead-of-time kernels at 8192 x 22016 (GPU box only): K0 quantize, K1
prepack, the fused quantize+pack, K3 de-quantise and unpack, each timed with
CUDA events (median of 5 after a warm-up) against its algorithmic HBM bytes
and MEASURED_PEAKS hbm_gbs.

env: KM, KK (shape), KE/KMB (format)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402

dev = torch.device("cuda:0")
M, K = int(os.environ.get("KM", 8192)), int(os.environ.get("KK", 22016))
fmt = fpx.FpxFormat(int(os.environ.get("KE", 3)), int(os.environ.get("KMB", 2)))
bits = fmt.total_bits
try:
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    peak = 6650.0
w32 = torch.randn(M, K, device=dev) * 0.02
w16 = w32.half()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


q = fpx.quantize_matrix(w32, fmt)
p = fpx.pack(q)
packed = M * K * bits / 8
rows = []
for name, fn, nbytes in [
    ("quantize fp32 (K0)", lambda: fpx.quantize_matrix(w32, fmt), M * K * 4 + M * K),
    ("quantize fp16 (K0)", lambda: fpx.quantize_matrix(w16, fmt), M * K * 2 + M * K),
    ("prepack (K1)", lambda: fpx.pack(q), M * K + packed),
    ("quantize+pack fused fp32", lambda: fpx.quantize_pack(w32, fmt), 2 * M * K * 4 + packed),
    ("quantize+pack fused fp16", lambda: fpx.quantize_pack(w16, fmt), 2 * M * K * 2 + packed),
    ("dequantize (K3)", lambda: fpx.dequantize(p), packed + 2 * M * K),
    ("unpack", lambda: fpx.unpack(p), packed + M * K),
]:
    us = timed(fn)
    gbs = nbytes / us / 1e3
    rows.append((name, us, nbytes, gbs))
    print(f"{name:28s} {us:9.1f} us  {nbytes / 1e6:8.1f} MB  {gbs:7.0f} GB/s  {gbs / peak:5.2f} of {peak:.0f}", flush=True)
