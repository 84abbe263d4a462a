"""Classic (N > 32) kernel correctness probe across batch / split / grid (GPU box only)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402

dev = torch.device("cuda:0")
M, K = int(os.environ.get("KM", 8192)), int(os.environ.get("KK", 22016))
p = fpx.pack(fpx.quantize_matrix(torch.randn(M, K, device=dev) * 0.02, fpx.FpxFormat.e3m2()))
W = fpx.dequantize(p).float()
for n in [int(x) for x in os.environ.get("NS", "64,128,256").split(",")]:
    act = torch.randn(n, K, device=dev).half()
    ref = act.float() @ W.t()
    for split in [int(x) for x in os.environ.get("SPLITS", "2,9").split(",")]:
        for grid in os.environ.get("GRIDS", "148,1000").split(","):
            os.environ["FPX_LINEAR_GRID"] = grid
            out = fpx.gemm_packed(p, act, split_k=split)
            err = float(((out - ref).abs().amax(dim=1) / ref.abs().amax(dim=1)).max())
            print(f"n={n} split={split} grid={grid} err={err:.2e}", flush=True)
