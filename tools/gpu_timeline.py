"""Whole-grid timeline of the decode kernel (GPU box only, bring-up tool).

Loads the tracing build (make -C paper_2401_14112_b200 trace) and prints,
per launch, the globaltimer events every CTA records (us, relative to the
earliest kernel entry): entry, prologue done, first weight stage landed,
unit ends, MMA issuer done, final barrier, exit -- as min / median / max over
CTAs -- for (a) an isolated launch (a spin kernel drains first) and (b) two
back-to-back launches with programmatic dependent launch (PDL).

env: KM, KK (shape), KN (batch), KSPLIT (split_k, 0 = default)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPX_B200_LIB", os.path.join(ROOT, "paper_2401_14112_b200", "libfpx_b200_trace.so"))
mode = os.environ.setdefault("FPX_LINEAR_TRACE", "2")
import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402

dev = torch.device("cuda:0")
L = fpx._lib.load()
M, K = int(os.environ.get("KM", 8192)), int(os.environ.get("KK", 22016))
n = int(os.environ.get("KN", 16))
split = int(os.environ.get("KSPLIT", 0)) or fpx.default_split(M, K, n)
fmt = fpx.FpxFormat.e3m2()
copies = [fpx.pack(fpx.quantize_matrix(torch.randn(M, K, device=dev) * 0.02, fmt)) for _ in range(3)]
ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
act = torch.randn(n, K, device=dev).half()
out = torch.empty(n, M, device=dev)
s = torch.cuda.current_stream().cuda_stream
EV = [("entry", 15), ("prologue", 0), ("data0", 14), ("unit1", 1), ("unit2", 2), ("unit3", 3), ("mma_done", 9),
      ("epi_done", 11), ("barrier", 7), ("exit", 13)]


def launch(i):
    p = copies[i % 3]
    ptrs = (C.c_void_p * 2)(*[t.data_ptr() for t in p.streams])
    st = L.fpx_linear(ptrs, 2, p.scales.data_ptr(), M, K, 3, 2, act.data_ptr(), K, n, out.data_ptr(), M, split,
                      ws.data_ptr(), ws.numel(), s)
    assert st == 0, L.fpx_last_error()


def grid_table(buf):
    cta = buf[12 * 512: 12 * 512 + 256 * 16].reshape(256, 16).astype(np.int64)
    return cta[cta[:, 15] > 0]


def report(name, tabs, base):
    print(f"== {name}")
    for ti, cta in enumerate(tabs):
        rel = np.where(cta > 0, (cta - base) / 1e3, np.nan)
        print(f"  launch {ti}: {len(cta)} CTAs")
        for ev, slot in EV:
            col = rel[:, slot]
            if np.all(np.isnan(col)):
                continue
            print(f"    {ev:>9s}: min {np.nanmin(col):7.2f}  median {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f} us")


for i in range(4):
    launch(i)
torch.cuda.synchronize()
buf = np.zeros(2 * 32 * 512, np.uint64)
# (a) isolated: spin first, one launch
for rep in range(3):
    torch.cuda._sleep(200000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launch(rep)
    e1.record()
    torch.cuda.synchronize()
    assert L.fpx_debug_trace(buf.ctypes.data, buf.size) == 0
    both = [grid_table(buf[:32 * 512]), grid_table(buf[32 * 512:])]
    # the newest launch is the buffer with the later entry stamps
    tab = max(both, key=lambda t: t[:, 15].max() if len(t) else 0)
    print(f"isolated rep {rep}: events {e0.elapsed_time(e1) * 1e3:.1f} us")
    report("isolated", [tab], tab[:, 15].min())
# (b) back-to-back pair under PDL: A then B, traced into the two buffers
torch.cuda._sleep(200000)
launch(0)
launch(1)
torch.cuda.synchronize()
assert L.fpx_debug_trace(buf.ctypes.data, buf.size) == 0
a, b = grid_table(buf[:32 * 512]), grid_table(buf[32 * 512:])
if a[:, 15].min() > b[:, 15].min():
    a, b = b, a
report("back-to-back pair (PDL)", [a, b], a[:, 15].min())
print("split", split, "n", n, "M", M, "K", K)
