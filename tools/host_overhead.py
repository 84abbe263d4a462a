"""Host-side cost of one fpx_linear call (GPU box only): wall time per call of
N asynchronous launches (the device queue absorbs them), against a trivial
C-ABI call for the ctypes floor."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_14112_b200 as fpx  # noqa: E402

dev = torch.device("cuda:0")
L = fpx._lib.load()
M, K, n = 8192, 22016, 16
p = fpx.quantize_pack(torch.randn(M, K, device=dev) * 0.02, fpx.FpxFormat.e3m2())
ptrs = (C.c_void_p * 2)(*[s.data_ptr() for s in p.streams])
split = fpx.default_split(M, K, n)
ws = torch.zeros(int(L.fpx_linear_workspace_size(M, K, K, n, split)), dtype=torch.uint8, device=dev)
act = torch.randn(n, K, device=dev).half()
out = torch.empty(n, M, device=dev)
s = torch.cuda.current_stream().cuda_stream
args = (ptrs, 2, p.scales.data_ptr(), M, K, 3, 2, act.data_ptr(), K, n, out.data_ptr(), M, split, ws.data_ptr(),
        ws.numel(), s)
for _ in range(20):
    L.fpx_linear(*args)
torch.cuda.synchronize()
for reps in (50, 200):
    t = time.perf_counter()
    for _ in range(reps):
        L.fpx_linear(*args)
    dt = (time.perf_counter() - t) / reps * 1e6
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        L.fpx_linear_default_split(M, K, n)
    dt0 = (time.perf_counter() - t) / reps * 1e6
    print(f"{reps} calls: fpx_linear {dt:.1f} us/call on the host, trivial C-ABI call {dt0:.2f} us")
