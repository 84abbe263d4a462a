"""Wall time of the Python API calls (quantize_matrix, pack, dequantize, unpack,
quantize_pack) and of the raw C-ABI prepack with / without the scale check,
plus a torch.profiler table (GPU box only).  Found the ~0.4 ms per-call
cudaMallocAsync remap fixed by the library-owned scratch pool."""
import time, torch, ctypes as C, sys
sys.path.insert(0, '.')
import paper_2401_14112_b200 as fpx
from paper_2401_14112_b200 import _lib
dev = torch.device('cuda:0')
M, K = 8192, 22016
fmt = fpx.FpxFormat(3, 2)
w = torch.randn(M, K, device=dev) * 0.02
q = fpx.quantize_matrix(w, fmt)
p = fpx.pack(q)
L = _lib.load()
def wall(fn, n=10):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6
wid = (C.c_int * 2)(*p.split.widths)
ptrs = (C.c_void_p * 2)(*[s.data_ptr() for s in p.streams])
st = torch.cuda.current_stream().cuda_stream
print("pack()            %.1f us" % wall(lambda: fpx.pack(q)))
print("fpx_prepack scales %.1f us" % wall(lambda: L.fpx_prepack(q.codes.data_ptr(), q.scales.data_ptr(), q.rows, q.cols, 3, 2, wid, 2, ptrs, st)))
print("fpx_prepack noscal %.1f us" % wall(lambda: L.fpx_prepack(q.codes.data_ptr(), None, q.rows, q.cols, 3, 2, wid, 2, ptrs, st)))
print("torch.empty x2     %.1f us" % wall(lambda: [torch.empty(L.fpx_stream_bytes(q.rows, q.cols, x), dtype=torch.uint8, device=dev) for x in (2, 4)]))
print("quantize_matrix    %.1f us" % wall(lambda: fpx.quantize_matrix(w, fmt)))
print("dequantize         %.1f us" % wall(lambda: fpx.dequantize(p)))
print("unpack             %.1f us" % wall(lambda: fpx.unpack(p)))
print("quantize_pack      %.1f us" % wall(lambda: fpx.quantize_pack(w, fmt)))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3): fpx.pack(q); fpx.dequantize(p); fpx.unpack(p); fpx.quantize_matrix(w, fmt)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
