"""Soak test (GPU box only): CUDA graphs of 60 back-to-back linears over three
rotated weight copies, replayed REPS times, for every routed batch width and
the three fused formats at default and forced splits; every output compared
bit for bit with a single reference launch.  Prints one line per case and
`soak ok` at the end; run it under `timeout` (a hang is the failure mode it
hunts).  env: REPS (50), KM / KK (weight shape, 4096 x 6144), NS (batch widths)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402

dev = torch.device("cuda:0")
reps = int(os.environ.get("REPS", 50))
KM, KK = int(os.environ.get("KM", 4096)), int(os.environ.get("KK", 6144))
NS = [int(x) for x in os.environ.get("NS", "1,7,16,17,32,48,64,100,128,200").split(",")]
total = 0
t0 = time.time()
for (e, m) in ((3, 2), (2, 3), (2, 2)):
    torch.manual_seed(e * 10 + m)
    p0 = fpx.quantize_pack(torch.randn(KM, KK, device=dev) * 0.02, fpx.FpxFormat(e, m))
    copies = [p0] + [fpx.PackedWeights(p0.format, p0.split, p0.rows, p0.cols, p0.orig_rows, p0.orig_cols,
                                       [s.clone() for s in p0.streams], p0.scales.clone()) for _ in range(2)]
    for n in NS:
        for sk in (0, 3, 7):
            x = torch.randn(n, p0.cols, device=dev).half()
            ref = fpx.gemm_packed(p0, x, split_k=sk)
            outs = [torch.full((n, p0.rows), float("nan"), device=dev) for _ in range(3)]
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(60):
                    fpx.gemm_packed(copies[i % 3], x, split_k=sk, out=outs[i % 3])
            for _ in range(reps):
                g.replay()
            torch.cuda.synchronize()
            bad = [i for i, o in enumerate(outs) if not torch.equal(o, ref)]
            total += 60 * reps
            print(f"e{e}m{m} n={n:3d} split_k={sk}: {60 * reps} launches, mismatching copies {bad}", flush=True)
            assert not bad
            del g
print(f"soak ok: {total} launches in {time.time() - t0:.0f} s")
