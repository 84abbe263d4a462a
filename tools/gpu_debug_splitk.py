"""Debug probe for split-K: dumps per-chunk partials, counters and C."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402
from paper_2401_14112_b200 import fpx as F  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402

O = Oracle()
dev = torch.device("cuda:0")
rng = np.random.default_rng(1)
e, m = 3, 2
M, K = 1024, 2048
w = (rng.standard_normal((M, K)) * 0.02).astype(np.float32)
st, c_o, s_o, _ = O.quantize(w, e, m)
p = fpx.pack(fpx.quantize_matrix(torch.from_numpy(w).to(dev), fpx.FpxFormat(e, m)))
W = O.dequantize(c_o, s_o, e, m).view(np.float16).astype(np.float64)
for n in [1, 16]:
    b = rng.standard_normal((n, K)).astype(np.float16)
    B = b.astype(np.float64)
    ref = B @ W.T  # [n, M]
    for S in [2, 5]:
        for rep in range(3):
            c = fpx.gemm_packed(p, torch.from_numpy(b).to(dev), split_k=S)
            torch.cuda.synchronize()
            ws = F._ws[(0, torch.cuda.current_stream(dev).cuda_stream)]
            cnt = ws[: 64 * 1024].view(torch.int32).cpu().numpy()
            part = ws[64 * 1024:].view(torch.float32).cpu().numpy()
            cg = c.cpu().numpy()
            rel = (np.abs(cg - ref).max(axis=1) / np.abs(ref).max(axis=1)).max()
            kt = K // 64
            tiles_m = M // 128
            npad = 16 if n <= 16 else 32
            bad_parts = []
            for mt in range(tiles_m):
                for ch in range(S):
                    k0, k1 = ch * kt // S * 64, (ch + 1) * kt // S * 64
                    exp = B[:, k0:k1] @ W[mt * 128:(mt + 1) * 128, k0:k1].T  # [n, 128]
                    off = (mt * S + ch) * npad * 128
                    got = part[off: off + npad * 128].reshape(npad, 128)[:n]
                    err = np.abs(got - exp).max() / max(np.abs(exp).max(), 1e-9)
                    if err > 1e-3:
                        bad_parts.append((mt, ch, float(err)))
            bad_rows = np.where(np.abs(cg - ref).max(axis=0) > 1e-3 * np.abs(ref).max())[0]
            print(f"n={n} S={S} rep={rep} relerr={rel:.3g} nonzero_counters={int((cnt != 0).sum())} "
                  f"bad_partials={bad_parts[:6]} nbad={len(bad_parts)} bad_rows={bad_rows[:10]} "
                  f"nbadrows={len(bad_rows)}", flush=True)
