"""Bring-up timing of fpx_linear pipeline variants (FPX_LINEAR_DBG knobs)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402

dev = torch.device("cuda:0")
L = fpx._lib.load()
M, K = int(os.environ.get("KM", 8192)), int(os.environ.get("KK", 22016))
fmt = fpx.FpxFormat.e3m2()
p0 = fpx.pack(fpx.quantize_matrix(torch.randn(M, K, device=dev) * 0.02, fmt))
copies = [p0] + [fpx.PackedWeights(p0.format, p0.split, p0.rows, p0.cols, p0.orig_rows, p0.orig_cols,
                                   [s.clone() for s in p0.streams], p0.scales.clone()) for _ in range(2)]
ptrs = [(C.c_void_p * 2)(*[s.data_ptr() for s in cp.streams]) for cp in copies]
ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream()
wbytes = M * K * 0.75


def timeit(n, split, iters=30):
    act = torch.randn(n, K, device=dev).half()
    out = torch.empty(n, M, device=dev)

    def go(i):
        cp = copies[i % 3]
        st = L.fpx_linear(ptrs[i % 3], 2, cp.scales.data_ptr(), M, K, 3, 2, act.data_ptr(), K, n, out.data_ptr(), M,
                          split, ws.data_ptr(), ws.numel(), stream.cuda_stream)
        assert st == 0, L.fpx_last_error()

    for i in range(5):
        go(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for i in range(iters):
        go(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / iters


# memcpy reference: read 3 x weight-size rotating buffers
src = [torch.empty(int(wbytes), dtype=torch.uint8, device=dev) for _ in range(3)]
dst = torch.empty(int(wbytes), dtype=torch.uint8, device=dev)
for i in range(3):
    dst.copy_(src[i])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for i in range(30):
    dst.copy_(src[i % 3])
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1000 / 30
print(f"torch copy of {wbytes/1e6:.0f} MB: {us:.1f} us  -> read+write {2*wbytes/us/1e3:.0f} GB/s", flush=True)

variants = os.environ.get("VARIANTS", "0,1,2,3,4,8,12,7,11").split(",")
cfgs = os.environ.get("CFGS", "").split(";") if os.environ.get("CFGS") else [None]
splits = [int(x) for x in os.environ.get("SPLITS", "1,2,4,9,23").split(",")]
ns = [int(x) for x in os.environ.get("NS", "1,16").split(",")]
for cfg in cfgs:
    if cfg:
        os.environ["FPX_LINEAR_CFG"] = cfg
    for n in ns:
        for split in splits:
            row = []
            for v in variants:
                os.environ["FPX_LINEAR_DBG"] = v
                row.append(f"dbg{v}={timeit(n, split):7.1f}")
            os.environ.pop("FPX_LINEAR_DBG", None)
            print(f"cfg={cfg} n={n:3d} split={split:2d} " + " ".join(row), flush=True)
