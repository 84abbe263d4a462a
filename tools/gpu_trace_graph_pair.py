"""Per-CTA timelines of two consecutive fpx_linear launches inside a CUDA graph
replay (GPU box only): the gap between one launch's last CTA exit and the next
launch's first CTA start.  FPX_LINEAR_TRACE=2 alternates trace buffers per call."""
import os
import sys

import numpy as np

os.environ["FPX_LINEAR_TRACE"] = "2"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPX_B200_LIB", os.path.join(ROOT, "paper_2401_14112_b200", "libfpx_b200_trace.so"))  # make ... trace
import torch  # noqa: E402

exec(open(os.path.join(ROOT, "tools", "gpu_prof_one.py")).read().split("for _ in range(int(os.environ")[0])


def go():
    st = L.fpx_linear(ptrs, 2, p.scales.data_ptr(), M, K, fmt.exp_bits, fmt.man_bits, act.data_ptr(), K, n,
                      out.data_ptr(), M, split, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    assert st == 0


for _ in range(2):
    go()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(10):
        go()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph: {e0.elapsed_time(e1) * 100:.2f} us per launch")
buf = np.zeros(2 * 32 * 512, np.uint64)
assert L.fpx_debug_trace(buf.ctypes.data, buf.size) == 0
tl = []
for b in range(2):
    c = buf[b * 16384 + 12 * 512: b * 16384 + 12 * 512 + 256 * 16].reshape(256, 16).astype(np.int64)
    tl.append(c[c[:, 0] > 0])
order = sorted(range(2), key=lambda b: tl[b][:, 0].min())
a, b = tl[order[0]], tl[order[1]]
base = a[:, 0].min()
for name, c in (("first", a), ("second", b)):
    r = (c - base) / 1e3
    print(f"{name}: start min/max {r[:, 0].min():.2f}/{r[:, 0].max():.2f}  teardown min/med/max "
          f"{r[:, 12].min():.2f}/{np.median(r[:, 12]):.2f}/{r[:, 12].max():.2f} us")
r = (a - base) / 1e3
names = {9: "mma", 14: "epi fence", 15: "epi atomic", 10: "red fence", 8: "red done", 11: "epilogue", 12: "all warps", 13: "tmem freed"}
for e, nm in names.items():
    v = np.where(a[:, e] > 0, r[:, e], np.nan)
    print(f"  {nm:12s} done: median {np.nanmedian(v):6.2f}  max {np.nanmax(v):6.2f} us (n={int(np.sum(a[:, e] > 0))})")
slow = int(np.argmax(r[:, 11]))
print("  slowest epilogue CTA:", " ".join(f"{k}={r[slow, k]:.2f}" for k in (1, 2, 3, 4, 14, 15, 10, 8, 11)))
print("  last unit end: median %.2f max %.2f" % (np.median(np.nanmax(np.where(a[:, 1:7] > 0, r[:, 1:7], np.nan), axis=1)),
                                              np.max(np.nanmax(np.where(a[:, 1:7] > 0, r[:, 1:7], np.nan), axis=1))))
print("gap last TMEM free -> next first start: %.2f us; period: %.2f us" % ((b[:, 0].min() - a[:, 13].max()) / 1e3,
                                                                       (b[:, 0].min() - a[:, 0].min()) / 1e3))
