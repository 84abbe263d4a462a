#!/usr/bin/env python3
"""Generate tests/golden/ from the UNMODIFIED reference library.

Runs in the builder container only (needs oracle/_ref/libfpxref.so, built by
`make -C oracle` from /root/reference/proj).  Writes:

  golden.npz   small cases (inputs are regenerated from the recorded seed):
               codes, scales, streams, dequantised fp16 W, gemm_reference C
  golden.json  scalar known-answer tables (decode / encode / effective_scale
               / half_mul samples) and FNV-1a-64 pins of full-size cases
               (4096^2 and llama-65b 8192x22016) whose arrays are too big to
               commit.

Inputs are numpy default_rng(seed).standard_normal(..., float32) * 0.02 for
weights and default_rng(seed+1).standard_normal(...).astype(float16) for
activations (col-major K x N stored as [N, K]); see `weights()` /
`activations()` -- the tests use the same functions.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, Reference, split_for  # noqa: E402

FORMATS = [(3, 2), (2, 3), (2, 2)]
SMALL = [  # (seed, rows, cols, batches)
    (1, 128, 128, (1, 8)),
    (2, 100, 200, (3,)),
    (3, 64, 64, (16,)),
    (4, 192, 320, (1, 32)),
]
FULL = [(11, 4096, 4096), (12, 8192, 22016)]


def weights(seed: int, rows: int, cols: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((rows, cols), dtype=np.float32) * np.float32(0.02)


def activations(seed: int, n: int, k: int) -> np.ndarray:
    return np.random.default_rng(seed + 1000).standard_normal((n, k), dtype=np.float32).astype(np.float16)


def fnv(o: Oracle, *arrs) -> str:
    return o.fnv1a64(*arrs)


def main():
    R, O = Reference(), Oracle()
    out = {}
    meta = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj (unmodified)",
            "weights": "default_rng(seed).standard_normal(float32) * 0.02",
            "activations": "default_rng(seed + 1000).standard_normal(float32).astype(float16), [N, K]",
            "cases": [], "full": [], "kat": {}}
    # ---- scalar KATs
    for e, m in FORMATS + [(2, 1), (4, 3), (3, 1), (5, 2), (4, 1), (1, 2)]:
        name = f"e{e}m{m}"
        codes = list(range(1 << (1 + e + m)))
        meta["kat"][name] = {
            "decode": [float(R.lib.ref_decode(c, e, m)) for c in codes],
            "encode_roundtrip": [int(R.lib.ref_encode(float(R.lib.ref_decode(c, e, m)), e, m)) for c in codes],
            "effective_scale": {str(s): int(R.lib.ref_effective_scale(s, e, m))
                                for s in (0x0001, 0x03ff, 0x0400, 0x3c00, 0x3800, 0x4200, 0x4bff, 0x2c00, 0x8001)},
        }
    rng = np.random.default_rng(99)
    vals = np.concatenate([rng.standard_normal(64).astype(np.float64) * 10.0, [1000.0, -0.0, 0.0, 28.0, 27.9, 0.03125,
                                                                               0.0625, 7.49, 7.5, -1e-9]])
    meta["kat"]["encode_samples"] = {f"e{e}m{m}": [[float(v), int(R.lib.ref_encode(float(v), e, m))] for v in vals]
                                     for e, m in FORMATS}
    hm = rng.integers(0, 1 << 16, size=(256, 2))
    meta["kat"]["half_mul"] = [[int(a), int(b), int(R.lib.ref_half_mul(int(a), int(b)))] for a, b in hm]
    # ---- small matrix cases
    for e, m in FORMATS:
        for seed, rows, cols, batches in SMALL:
            tag = f"e{e}m{m}_{rows}x{cols}_s{seed}"
            w = weights(seed, rows, cols)
            st, codes, scales = R.quantize(w, e, m)
            assert st == 0, R.last_error()
            st, streams = R.pack(codes, scales, e, m, rows, cols)
            assert st == 0, R.last_error()
            st, deq = R.dequantize(codes, scales, e, m)
            assert st == 0
            out[f"{tag}/codes"] = codes
            out[f"{tag}/scales"] = scales
            for i, s in enumerate(streams):
                out[f"{tag}/stream{i}"] = s
            out[f"{tag}/dequant"] = deq
            h = R.prepare(codes, scales, e, m, rows, cols)
            for n in batches:
                b = activations(seed, n, cols).view(np.uint16)
                out[f"{tag}/C_n{n}"] = h.gemm_reference(b)
                cp = h.gemm_packed(b)
                assert (cp.view(np.uint32) == out[f"{tag}/C_n{n}"].view(np.uint32)).all()
            meta["cases"].append({"tag": tag, "e": e, "m": m, "seed": seed, "rows": rows, "cols": cols,
                                  "batches": list(batches), "split": split_for(e, m)})
            print("case", tag, flush=True)
    # ---- full-size pins (hashes only)
    for seed, rows, cols in FULL:
        w = weights(seed, rows, cols)
        for e, m in FORMATS if rows == 8192 else [(3, 2)]:
            st, codes, scales = R.quantize(w, e, m)
            assert st == 0
            st, streams = R.pack(codes, scales, e, m, rows, cols)
            assert st == 0
            meta["full"].append({"seed": seed, "rows": rows, "cols": cols, "e": e, "m": m,
                                 "codes_fnv": fnv(O, codes), "scales_fnv": fnv(O, scales),
                                 "streams_fnv": [fnv(O, s) for s in streams]})
            print("full", seed, rows, cols, e, m, flush=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", os.path.join(HERE, "golden.npz"), os.path.getsize(os.path.join(HERE, "golden.npz")))


if __name__ == "__main__":
    main()
