"""Step-by-step GPU bring-up probe (prints, does not assert).

Run on the GPU box:  timeout 300 python tools/gpu_probe.py
Each stage compares the sm_100a kernels with the C oracle and prints the
mismatch statistics, so a failing stage can be diagnosed from one run.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

O = Oracle()
dev = torch.device("cuda:0")
print("device", torch.cuda.get_device_name(0), torch.cuda.get_device_capability(0), flush=True)


def u16(t):
    return t.cpu().numpy().view(np.uint16)


def stage(name):
    print(f"\n=== {name}", flush=True)


rng = np.random.default_rng(1)
for (e, m) in [(3, 2), (2, 3), (2, 2)]:
    fmt = fpx.FpxFormat(e, m)
    stage(f"quantize/pack/dequant {fmt.name()}")
    w = (rng.standard_normal((200, 300)) * 0.02).astype(np.float32)
    st, c_o, s_o, _ = O.quantize(w, e, m)
    q = fpx.quantize_matrix(torch.from_numpy(w).to(dev), fmt)
    torch.cuda.synchronize()
    print("codes equal", bool((q.codes.cpu().numpy() == c_o).all()), "scales equal",
          bool((u16(q.scales) == s_o).all()))
    p = fpx.pack(q)
    _, st_o = O.pack(c_o, s_o, e, m)
    for i, (a, b) in enumerate(zip(p.streams, st_o)):
        print(f"stream{i} equal", bool((a.cpu().numpy() == b).all()))
    u = fpx.unpack(p)
    print("unpack roundtrip", bool((u.codes.cpu().numpy() == c_o).all()))
    d = fpx.dequantize(p)
    d_o = O.dequantize(c_o, s_o, e, m)
    dd = u16(d)
    bad = (dd != d_o)
    print("dequant mismatches", int(bad.sum()), "of", bad.size)
    if bad.any():
        idx = np.argwhere(bad)[:5]
        for r, c in idx:
            print("  at", r, c, "gpu %04x oracle %04x code %d scale %04x" % (dd[r, c], d_o[r, c], c_o[r, c], s_o[r]))

    stage(f"linear {fmt.name()}")
    for n in [1, 8, 16, 32, 100]:
        b = (rng.standard_normal((n, 300))).astype(np.float16)
        _, c_ref = O.gemm_reference(c_o, s_o, e, m, b.view(np.uint16), orig_cols=300)
        t0 = time.time()
        try:
            c = fpx.gemm_packed(p, torch.from_numpy(b).to(dev))
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001
            print("n", n, "FAILED", ex)
            continue
        cg = c.cpu().numpy()
        err = np.abs(cg - c_ref).max(axis=1)
        nrm = np.abs(c_ref).max(axis=1)
        print("n", n, "max rel err per vector", float((err / np.maximum(nrm, 1e-30)).max()), "time", time.time() - t0)
        if not np.isfinite(cg).all():
            print("  non-finite outputs", int((~np.isfinite(cg)).sum()))
        if (err / np.maximum(nrm, 1e-30)).max() > 1e-2:
            j = int(np.argmax(err / np.maximum(nrm, 1e-30)))
            r = np.argsort(-np.abs(cg[j] - c_ref[j]))[:8]
            print("  worst vector", j, "rows", r, "gpu", cg[j, r], "ref", c_ref[j, r])

stage("linear larger shapes / split-K")
e, m = 3, 2
fmt = fpx.FpxFormat(e, m)
w = (rng.standard_normal((1024, 2048)) * 0.02).astype(np.float32)
st, c_o, s_o, _ = O.quantize(w, e, m)
p = fpx.pack(fpx.quantize_matrix(torch.from_numpy(w).to(dev), fmt))
for n in [1, 16, 32]:
    b = (rng.standard_normal((n, 2048))).astype(np.float16)
    _, c_ref = O.gemm_reference(c_o, s_o, e, m, b.view(np.uint16))
    outs = {}
    for sk in [1, 2, 5, 32]:
        c = fpx.gemm_packed(p, torch.from_numpy(b).to(dev), split_k=sk)
        torch.cuda.synchronize()
        cg = c.cpu().numpy()
        outs[sk] = cg
        err = np.abs(cg - c_ref).max(axis=1) / np.maximum(np.abs(c_ref).max(axis=1), 1e-30)
        print("n", n, "split", sk, "max rel err", float(err.max()))
    os.environ["FPX_LINEAR_GRID"] = "7"
    c7 = fpx.gemm_packed(p, torch.from_numpy(b).to(dev), split_k=5).cpu().numpy()
    del os.environ["FPX_LINEAR_GRID"]
    print("  grid-independence (split 5, grid 7 vs 148) bit-equal:", bool((c7.view(np.uint32) == outs[5].view(np.uint32)).all()))

stage("timing 8192x22016 e3m2")
M, K = 8192, 22016
wt = torch.randn(M, K, device=dev) * 0.02
q = fpx.quantize_matrix(wt, fmt)
p = fpx.pack(q)
del wt, q
for n in [1, 8, 16, 32, 128]:
    b = torch.randn(n, K, device=dev).half()
    for _ in range(3):
        fpx.gemm_packed(p, b)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    iters = 20
    for _ in range(iters):
        fpx.gemm_packed(p, b)
    ev1.record()
    torch.cuda.synchronize()
    us = ev0.elapsed_time(ev1) * 1000 / iters
    print(f"n {n}: {us:.1f} us  weight GB/s {M * K * 0.75 / us / 1e3:.0f}", flush=True)
print("done")
