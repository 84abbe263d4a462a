"""Print CTA 0's per-stage pipeline timeline of one fpx_linear launch.

Run with FPX_LINEAR_TRACE=1 (env KM/KK/KN/KS as gpu_prof_one.py)."""
import os
import sys

import numpy as np

os.environ["FPX_LINEAR_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPX_B200_LIB", os.path.join(ROOT, "paper_2401_14112_b200", "libfpx_b200_trace.so"))  # make ... trace
import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402

exec(open(os.path.join(ROOT, "tools", "gpu_prof_one.py")).read().split("for _ in range(int(os.environ")[0])
for _ in range(3):
    st = L.fpx_linear(ptrs, 2, p.scales.data_ptr(), M, K, fmt.exp_bits, fmt.man_bits, act.data_ptr(), K, n,
                      out.data_ptr(), M, split, ws.data_ptr(), ws.numel(), s)
torch.cuda.synchronize()
buf = np.zeros(16 * 512, np.uint64)
assert L.fpx_debug_trace(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(16, 512)[:10].astype(np.int64)
names = ["prod_issue", "dq_aempty", "dq_full", "dq_done", "mma_afull", "mma_issued", "epi_full(unit)"]
t0 = tr[0][tr[0] > 0].min()
ns = int((tr[0] > 0).sum())
print("split", split, "stages traced", ns)
print("stage " + " ".join(f"{x:>11s}" for x in names[:6]))
for si in range(min(ns, 80)):
    print(f"{si:5d} " + " ".join(f"{(tr[e][si] - t0) / 1.9e3:11.2f}" if tr[e][si] else f"{'-':>11s}" for e in range(6)))
print("epilogue unit arrivals (us):", [round((x - t0) / 1.9e3, 2) for x in tr[6] if x])
d = lambda a, b: (tr[b][:ns] - tr[a][:ns]) / 1.9e3  # noqa: E731
ok = (tr[1][:ns] > 0)
print("mean us: full-wait after aempty %.3f | dequant (full->done) %.3f | done->mma_afull %.3f | mma issue %.3f"
      % (np.mean(d(1, 2)[ok]), np.mean(d(2, 3)[ok]), np.mean(d(3, 4)[ok]), np.mean(d(4, 5)[ok])))
print("mean inter-stage (mma_issued) us: %.3f" % np.mean(np.diff(tr[5][:ns]) / 1.9e3))
print("load latency prod_issue->dq_full us: %.3f" % np.mean(d(0, 2)[ok]))
print("quarter done offsets vs q0 (us) mean q1 %.3f q2 %.3f q3 %.3f | max-quarter-done -> mma_afull %.3f" % (
    np.mean(d(3, 7)[ok]), np.mean(d(3, 8)[ok]), np.mean(d(3, 9)[ok]),
    np.mean((tr[4][:ns] - np.maximum.reduce([tr[3][:ns], tr[7][:ns], tr[8][:ns], tr[9][:ns]]))[ok]) / 1.9e3))
for si in range(40, min(ns, 56)):
    print(si, " ".join(f"{(tr[e][si] - t0) / 1.9e3:7.2f}" for e in (2, 3, 7, 8, 9, 4, 5)))
