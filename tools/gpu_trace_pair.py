"""Per-CTA timelines of two consecutive fpx_linear launches (GPU box only):
how long the second launch's CTAs wait after the first launch's CTAs exit.
FPX_LINEAR_TRACE=2 is set here; env KM/KK/KN/KS as gpu_prof_one.py."""
import os
import sys

import numpy as np

os.environ["FPX_LINEAR_TRACE"] = "2"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FPX_B200_LIB", os.path.join(ROOT, "paper_2401_14112_b200", "libfpx_b200_trace.so"))  # make ... trace
import torch  # noqa: E402

exec(open(os.path.join(ROOT, "tools", "gpu_prof_one.py")).read().split("for _ in range(int(os.environ")[0])
for _ in range(4):  # calls 0..3 -> buffers 0,1,0,1: the last two launches are consecutive
    st = L.fpx_linear(ptrs, 2, p.scales.data_ptr(), M, K, fmt.exp_bits, fmt.man_bits, act.data_ptr(), K, n,
                      out.data_ptr(), M, split, ws.data_ptr(), ws.numel(), s)
torch.cuda.synchronize()
buf = np.zeros(2 * 32 * 512, np.uint64)
assert L.fpx_debug_trace(buf.ctypes.data, buf.size) == 0
tl = []
for b in range(2):
    c = buf[b * 16384 + 12 * 512: b * 16384 + 12 * 512 + 256 * 16].reshape(256, 16).astype(np.int64)
    tl.append(c[c[:, 0] > 0])
base = tl[0][:, 0].min()
for b, c in enumerate(tl):
    r = (c - base) / 1e3
    r[c == 0] = np.nan
    print(f"launch {b}: CTAs {len(c)} start min/max {np.nanmin(r[:, 0]):.2f}/{np.nanmax(r[:, 0]):.2f} "
          f"exit min/median/max {np.nanmin(r[:, 7]):.2f}/{np.nanmedian(r[:, 7]):.2f}/{np.nanmax(r[:, 7]):.2f} us")
print("gap: last exit of launch 0 -> first start of launch 1: %.2f us" % ((tl[1][:, 0].min() - tl[0][:, 7].max()) / 1e3))
print("period (launch-0 first start -> launch-1 first start): %.2f us" % ((tl[1][:, 0].min() - tl[0][:, 0].min()) / 1e3))
