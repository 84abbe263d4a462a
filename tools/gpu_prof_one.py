"""Run one fpx_linear configuration a few times (for ncu captures).

env: KM, KK (shape), KN (batch), KS (split_k, 0 = default), ITERS."""
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
n, split = int(os.environ.get("KN", 1)), int(os.environ.get("KS", 0))
fmt = fpx.FpxFormat(int(os.environ.get("KE", 3)), int(os.environ.get("KMB", 2)))
p = fpx.pack(fpx.quantize_matrix(torch.randn(M, K, device=dev) * 0.02, fmt))
split = split or fpx.default_split(M, K, n)
ptrs = (C.c_void_p * 2)(*[s.data_ptr() for s in p.streams])
ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
act = torch.randn(n, K, device=dev).half()
out = torch.empty(n, M, device=dev)
s = torch.cuda.current_stream().cuda_stream
for _ in range(int(os.environ.get("ITERS", 4))):
    st = L.fpx_linear(ptrs, 2, p.scales.data_ptr(), M, K, fmt.exp_bits, fmt.man_bits, act.data_ptr(), K, n,
                      out.data_ptr(), M, split, ws.data_ptr(), ws.numel(), s)
    assert st == 0, L.fpx_last_error()
torch.cuda.synchronize()
print("ok split", split)
