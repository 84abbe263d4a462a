"""CTA 0 per-stage timeline of one grouped fpx_linear launch (GPU box only).

FPX_LINEAR_TRACE=1 is set here; env KM/KK/KN/KS as gpu_prof_one.py.
Columns (us from the first producer issue): producer issue, group start
(before full wait), full seen, k-tile-0 dequant done, slot free, named
barrier passed, last MMA issued."""
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
buf = np.zeros(32 * 512, np.uint64)
assert L.fpx_debug_trace(buf.ctypes.data, buf.size) == 0
tr = buf.reshape(32, 512).astype(np.int64)
ev = {"pwait": 9, "prod": 0, "start": 1, "full": 2, "dq0": 3, "slot": 7, "ready": 4, "mwait": 10, "mgo": 11, "mma": 5}
t0 = tr[0][tr[0] > 0].min()
ns = int((tr[0] > 0).sum())
clk = float(os.environ.get("CLK_GHZ", "1.9")) * 1e3
f = lambda e, si: (tr[ev[e]][si] - t0) / clk if tr[ev[e]][si] else float("nan")  # noqa: E731
print("split", split, "stages traced", ns, "epilogue unit arrivals (us):",
      [round((x - t0) / clk, 2) for x in tr[6] if x])
print("stage " + " ".join(f"{k:>8s}" for k in ev))
for si in range(min(ns, 120)):
    print(f"{si:5d} " + " ".join(f"{f(k, si):8.2f}" for k in ev))
d = lambda a, b: np.array([f(b, si) - f(a, si) for si in range(ns)])  # noqa: E731
for a, b in [("pwait", "prod"), ("prod", "full"), ("start", "full"), ("full", "dq0"), ("dq0", "slot"), ("slot", "ready"), ("mwait", "mgo"), ("mgo", "mma")]:
    x = d(a, b)
    print(f"mean {a:>5s} -> {b:<5s}: {np.nanmean(x):.3f} us")
print("mean inter-stage (prod issue): %.3f us" % np.nanmean(np.diff([f('prod', si) for si in range(ns)])))
print("mean MMA-thread loop body (issued -> next wait): %.3f us" % np.nanmean([f('mwait', si + 1) - f('mma', si) for si in range(ns - 1)]))
print("mean producer loop body (issue -> next pre-wait): %.3f us" % np.nanmean([f('pwait', si + 1) - f('prod', si) for si in range(ns - 1)]))

# whole-grid timeline (globaltimer, ns)
cta = buf[12 * 512: 12 * 512 + 256 * 16].reshape(256, 16).astype(np.int64)
live = cta[:, 0] > 0
cta = cta[live]
base = cta[:, 0].min()
rel = np.where(cta > 0, (cta - base) / 1e3, np.nan)
print(f"CTAs {len(cta)}: start spread {np.nanmax(rel[:, 0]):.2f} us; exit min/median/max "
      f"{np.nanmin(rel[:, 7]):.2f}/{np.nanmedian(rel[:, 7]):.2f}/{np.nanmax(rel[:, 7]):.2f} us")
nunits = np.sum(~np.isnan(rel[:, 1:7]), axis=1)
for k in sorted(set(nunits.tolist())):
    sel = nunits == k
    last = rel[sel, k] if k else rel[sel, 0]
    print(f"  {sel.sum():3d} CTAs with {k} units: last unit end mean {np.nanmean(last):.2f} max {np.nanmax(last):.2f} us;"
          f" unit durations mean {np.nanmean(np.diff(rel[sel, :k + 1], axis=1)):.2f} us")
slow = np.argsort(-rel[:, 7])[:5]
for i in slow:
    print("  slowest CTA", i, " ".join(f"{x:7.2f}" for x in rel[i]))
names = {15: "entry", 0: "prologue", 14: "1st wstage", 1: "unit1 epi", 9: "mma done", 11: "epi done", 7: "sync",
         12: "teardown", 13: "dealloc", 8: "exit"}
print("per-CTA event medians (us from the earliest prologue):",
      " ".join(f"{nm}={np.nanmedian(rel[:, k]):.2f}" for k, nm in names.items() if np.any(~np.isnan(rel[:, k]))))
