"""Bring-up timing sweep of fpx_linear pipeline variants (GPU box only).

env: KM/KK shape; NS batches; SPLITS; CFGS
("KS,G;..."); VARIANTS (FPX_LINEAR_DBG values: 1 no dequant, 2 no MMA,
4 no weight loads, 8 no activation loads).  Each timing is 30 back-to-back
launches over 3 rotated weight copies (405 MB > L2); every configuration is
also checked against dequantize() @ act within the parity tolerance."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

last_mhz = 0

import paper_2401_14112_b200 as fpx  # noqa: E402

dev = torch.device("cuda:0")
L = fpx._lib.load()
M, K = int(os.environ.get("KM", 8192)), int(os.environ.get("KK", 22016))
fmt = fpx.FpxFormat(int(os.environ.get("KE", 3)), int(os.environ.get("KMB", 2)))
p0 = fpx.pack(fpx.quantize_matrix(torch.randn(M, K, device=dev) * 0.02, fmt))
copies = [p0] + [fpx.PackedWeights(p0.format, p0.split, p0.rows, p0.cols, p0.orig_rows, p0.orig_cols,
                                   [s.clone() for s in p0.streams], p0.scales.clone()) for _ in range(2)]
ptrs = [(C.c_void_p * 2)(*[s.data_ptr() for s in cp.streams]) for cp in copies]
ws = torch.zeros(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream()
wbytes = M * K * fmt.total_bits / 8
W16 = fpx.dequantize(p0).float()


def run(n, split, act, out, i):
    cp = copies[i % 3]
    st = L.fpx_linear(ptrs[i % 3], 2, cp.scales.data_ptr(), M, K, fmt.exp_bits, fmt.man_bits, act.data_ptr(), K, n,
                      out.data_ptr(), M, split, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    assert st == 0, L.fpx_last_error()


class Clocks:
    """SM clock samples (NVML, ~1 ms) while a timing runs: power-capped
    clocks move the compute-bound variants."""

    def __init__(self):
        import threading
        import pynvml
        pynvml.nvmlInit()
        self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(0)
        self.samples, self.on, self.threading = [], False, threading

    def __enter__(self):
        self.samples, self.on = [], True

        def loop():
            while self.on:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
        self.t = self.threading.Thread(target=loop, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.on = False
        self.t.join()

    def median(self):
        return sorted(self.samples)[len(self.samples) // 2] if self.samples else 0


CLK = Clocks() if os.environ.get("CLOCKS") else None


def timeit(n, split, iters=int(os.environ.get("ITERS", 30))):
    """Device time per launch: `iters` launches captured in one CUDA graph and
    replayed (host launch overhead excluded; the plain launch loop is
    host-bound at ~20 us per call through ctypes)."""
    act = torch.randn(n, K, device=dev).half()
    out = torch.empty(n, M, device=dev)
    for i in range(3):
        run(n, split, act, out, i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(iters):
            run(n, split, act, out, i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    global last_mhz
    if CLK:
        with CLK:
            for _ in range(20):  # ~20 x iters launches: long enough to sample the clock under load
                g.replay()
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
        last_mhz = CLK.median()
    else:
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
    err = None
    if not os.environ.get("FPX_LINEAR_DBG"):
        run(n, split, act, out, 0)
        ref = act.float() @ W16.t()
        err = float(((out - ref).abs().amax(dim=1) / ref.abs().amax(dim=1)).max())
    return e0.elapsed_time(e1) * 1000 / iters, err


variants = os.environ.get("VARIANTS", "0").split(",")
cfgs = os.environ.get("CFGS", "").split(";") if os.environ.get("CFGS") else [None]
splits = [int(x) for x in os.environ.get("SPLITS", "0").split(",")]
ns = [int(x) for x in os.environ.get("NS", "1,16").split(",")]
print(f"M={M} K={K} {fmt.name()} weight bytes {wbytes/1e6:.1f} MB", flush=True)
for kern in ["decode"]:
    for cfg in cfgs:
        if cfg:
            os.environ["FPX_LINEAR_CFG"] = cfg
        else:
            os.environ.pop("FPX_LINEAR_CFG", None)
        for n in ns:
            for split in splits:
                sp = split or fpx.default_split(M, K, n)
                row = []
                for v in variants:
                    if v != "0":
                        os.environ["FPX_LINEAR_DBG"] = v
                    print(f"  .. {kern} cfg={cfg} n={n} split={sp} dbg{v}", flush=True)
                    us, err = timeit(n, sp)
                    os.environ.pop("FPX_LINEAR_DBG", None)
                    row.append(f"dbg{v}={us:6.1f}us({wbytes / us / 1e3:5.0f}GB/s)" + (f" err={err:.1e}" if err is not None else "")
                               + (f" {last_mhz}MHz" if CLK else ""))
                print(f"{kern:8s} cfg={cfg} n={n:3d} split={sp:2d} " + " ".join(row), flush=True)
