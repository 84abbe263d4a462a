"""Steady-state H2D / D2H bandwidth of the e2e step's copy sizes from pinned
host memory allocated several ways (GPU box only): torch pin_memory, mmap'd
memory registered with cudaHostRegister with and without transparent huge
pages (madvise MADV_HUGEPAGE), and cudaHostAlloc with each flag."""
import ctypes
import mmap
import sys

import torch

libc = ctypes.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = ctypes.c_void_p
libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_long]
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
MADV_HUGEPAGE = 14


def registered(nbytes, huge):
    size = (nbytes + (2 << 20) - 1) // (2 << 20) * (2 << 20) + (2 << 20)
    addr = libc.mmap(None, size, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    base = (addr + (2 << 20) - 1) // (2 << 20) * (2 << 20)
    if huge:
        libc.madvise(ctypes.c_void_p(base), size - (2 << 20), MADV_HUGEPAGE)
    buf = (ctypes.c_uint8 * nbytes).from_address(base)
    ctypes.memset(base, 1, nbytes)
    t = torch.frombuffer(buf, dtype=torch.uint8)
    r = torch.cuda.cudart().cudaHostRegister(base, nbytes, 0)
    assert int(r) == 0, r
    return t


def bw(h, d, reps=200):
    res = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(h.numel() * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1)
    return res


print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
for nb in (2_774_016, 2_064_384, 64 << 20):
    d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    h1 = torch.empty(nb, dtype=torch.uint8).pin_memory()
    print(f"{nb / 1e6:7.2f} MB torch pinned     ", bw(h1, d))
    print(f"{nb / 1e6:7.2f} MB registered 4K    ", bw(registered(nb, False), d))
    print(f"{nb / 1e6:7.2f} MB registered THP   ", bw(registered(nb, True), d))
sys.stdout.flush()

# cudaHostAlloc flag variants through the runtime torch itself loaded
import glob  # noqa: E402
import os  # noqa: E402

cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(cands[0]) if cands else ctypes.CDLL("libcudart.so")
rt.cudaHostAlloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
nb = 2_774_016
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
for flags, nm in ((0, "Default"), (1, "Portable"), (2, "Mapped"), (4, "WriteCombined")):
    p = ctypes.c_void_p()
    assert rt.cudaHostAlloc(ctypes.byref(p), nb, flags) == 0
    ctypes.memset(p.value, 1, nb)
    h = torch.frombuffer((ctypes.c_uint8 * nb).from_address(p.value), dtype=torch.uint8)
    print(f"cudaHostAlloc {nm:14s}", bw(h, d))
h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
print("torch.empty(pin_memory=True) ", bw(h, d))
h = torch.ones(nb, dtype=torch.uint8).pin_memory()
print("torch .pin_memory() (ones)   ", bw(h, d))
