#!/usr/bin/env python3
"""bench.py -- W6A16 (FP6 e3m2) linear on llama-65B FFN shapes, B200.

Workload (BASELINE.json configs[1]): weight 8192 x 22016 FP6 e3m2 with
per-row fp16 scales, one step = one fused linear (fpx_linear, the C-ABI hot
path) for each batch N in {1, 2, 4, 8, 16, 32} -- the "batch 1-32" sweep the
metric is quoted on.  Synthetic N(0, 0.02) weights (quantized + packed on the
GPU by our own kernels, bit-exact with the reference) and N(0, 1) fp16
activations; no checkpoints or datasets.

value  = whole-job weight-byte throughput (GB/s): sum over ranks and launches
         of M*K*6/8 bytes / max-over-ranks device time of the K timed steps.
L2     : every launch reads a different copy of the packed weights (3 copies
         rotated, 3 x 135 MB > 126 MB L2), so no launch hits weights left in
         L2 by the previous two.
e2e    : same sweep through the public API with host buffers: pinned host
         activations -> H2D, fpx_linear, C -> pinned host (D2H) every launch,
         copies on two copy streams pipelined against the launches; packed
         weights stay resident in HBM (loaded once, like a model).
--impl reference: the reference's own CPU gemm_packed (oracle/_ref, compiled
         unmodified from /root/reference) on the host cores, same workload.

Multi-GPU (torchrun): weak scaling -- every rank runs the full step on its
own weights (the path shards by independent output tiles; no data-path
collective), timings reduced with MAX over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M_ROWS, K_COLS = 8192, 22016
BATCHES = (1, 2, 4, 8, 16, 32)
METRIC = "W6A16 linear µs & achieved HBM GB/s (llama-65b shapes, batch 1–32)"
WEIGHT_BYTES = M_ROWS * K_COLS * 6 // 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batches", default=",".join(map(str, BATCHES)))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.time() + 5.0
            while not self.rows and time.time() < t_end:  # sampler is up before timing starts
                time.sleep(0.01)
            self.rows.clear()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "window": "timed region + 0.3 s of the identical step directly after (nvidia-smi -lms 20)"}


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of the decode kernel from the
    committed ncu --set full capture (profiles/), bytes per launch, or None."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_decode_n16_summary.txt")))
    if not files:
        return None, None
    txt = open(files[-1]).read()
    rd = re.search(r"dram__bytes_read.sum = ([0-9.]+) Mbyte", txt)
    wr = re.search(r"dram__bytes_write.sum = ([0-9.]+) Mbyte", txt)
    if not (rd and wr):
        return None, None
    return round((float(rd.group(1)) + float(wr.group(1))) * 1e6), os.path.relpath(files[-1], ROOT)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


# --------------------------------------------------------------------- ours
def run_ours(args, rank, world, local):
    import torch

    import paper_2401_14112_b200 as fpx
    from paper_2401_14112_b200 import fpx as F

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    batches = [int(x) for x in args.batches.split(",")]
    fmt = fpx.FpxFormat.e3m2()
    L = fpx._lib.load()

    # ---- setup (untimed): synthetic weights, quantize + pack on GPU
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    w = torch.randn(M_ROWS, K_COLS, device=dev, generator=g) * 0.02
    q = fpx.quantize_matrix(w, fmt)
    packed = fpx.pack(q)
    codes_host = q.codes.cpu().numpy() if (rank == 0 and not args.no_cpu_baseline) else None
    scales_host = q.scales.cpu().numpy().view(np.uint16) if codes_host is not None else None
    del w, q
    n_copies = 3
    copies = [packed] + [fpx.PackedWeights(packed.format, packed.split, packed.rows, packed.cols, packed.orig_rows,
                                           packed.orig_cols, [s.clone() for s in packed.streams],
                                           packed.scales.clone()) for _ in range(n_copies - 1)]
    acts = {n: (torch.randn(n, K_COLS, device=dev, generator=g)).half() for n in batches}
    outs = {n: torch.empty(n, M_ROWS, device=dev) for n in batches}
    splits = {n: fpx.default_split(M_ROWS, K_COLS, n) for n in batches}
    ws_need = max(int(L.fpx_linear_workspace_size(M_ROWS, K_COLS, K_COLS, n, splits[n])) for n in batches)
    ws = torch.zeros(ws_need, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    import ctypes as C
    ptrs = [(C.c_void_p * 2)(*[s.data_ptr() for s in cp.streams]) for cp in copies]

    def launch(i, n, act_ptr, out_ptr):
        cp = copies[i % n_copies]
        st = L.fpx_linear(ptrs[i % n_copies], 2, cp.scales.data_ptr(), M_ROWS, K_COLS, 3, 2, act_ptr, K_COLS, n,
                          out_ptr, M_ROWS, splits[n], ws.data_ptr(), ws.numel(),
                          torch.cuda.current_stream(dev).cuda_stream)
        if st:
            raise RuntimeError(L.fpx_last_error().decode())

    def step(counter):
        for n in batches:
            launch(counter, n, acts[n].data_ptr(), outs[n].data_ptr())
            counter += 1
        return counter

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def capture(fn):
        """CUDA graph of fn(): a decode step is ~0.2 ms of device work but ~0.15 ms of
        host-side ctypes/C-ABI calls, so eager launches would time the host."""
        torch.cuda.synchronize(dev)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        gr.replay()  # warm
        torch.cuda.synchronize(dev)
        return gr

    def timed(gr, reps=1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record()
        for _ in range(reps):
            gr.replay()
        e1.record()
        barrier()
        return e0.elapsed_time(e1)

    cnt = 0
    for _ in range(args.warmup):
        cnt = step(cnt)
    nl = len(batches) * args.steps
    state = {"cnt": cnt}

    def k_steps():
        c = state["cnt"]
        for _ in range(args.steps):
            c = step(c)

    # per-batch device time of the fused kernel (informational: graph of 12
    # launches per N, 3 weight copies rotated), measured before the timed
    # region and its clock soak
    per_n = {}
    for n in batches:
        gr = capture(lambda: [launch(i, n, acts[n].data_ptr(), outs[n].data_ptr()) for i in range(12)])
        per_n[n] = max_over_ranks(timed(gr, 2) * 1e3 / 24)  # us per launch

    g_steps = capture(k_steps)
    for _ in range(args.warmup):  # warm-up replays of the timed graph itself
        g_steps.replay()
    barrier()
    with ClockSampler(local) as clk:
        total_ms = max_over_ranks(timed(g_steps))
        # The timed region lasts a few ms, below nvidia-smi's sampling period:
        # keep replaying the identical steps (untimed) for >= 0.3 s so the
        # clock/throttle samples describe this workload under load.
        soak_end = time.time() + 0.3
        while time.time() < soak_end:
            g_steps.replay()
            torch.cuda.synchronize(dev)


    # ---- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # A step's activations (all six batches) live in ONE pinned host block and
        # ONE device block, and so do its outputs: one H2D and one D2H per step
        # (each small cudaMemcpy costs several us of copy-engine time).
        tot_a = sum(n * K_COLS for n in batches)
        tot_c = sum(n * M_ROWS for n in batches)
        h_act_all = torch.cat([acts[n].reshape(-1) for n in batches]).cpu().pin_memory()
        h_out_all = torch.empty(tot_c, pin_memory=True)

        def views(buf, per_row):
            out, off = {}, 0
            for n in batches:
                out[n] = buf[off: off + n * per_row].view(n, per_row)
                off += n * per_row
            return out

        # two device buffer sets (step parity), so step k+1's uploads overlap step k's compute
        d_act_all = [torch.empty(tot_a, dtype=torch.float16, device=dev) for _ in range(2)]
        d_out_all = [torch.empty(tot_c, dtype=torch.float32, device=dev) for _ in range(2)]
        d_act = [views(b, K_COLS) for b in d_act_all]
        d_out = [views(b, M_ROWS) for b in d_out_all]
        s_h2d = torch.cuda.Stream(dev)
        s_d2h = torch.cuda.Stream(dev)

        def e2e_steps():
            """Per step: the step's activations H2D on a copy stream, the six
            fused linears back to back on the compute stream (consecutive
            launches keep their programmatic-dependent-launch overlap), the
            six fp32 C D2H on a second copy stream (PCIe is full duplex).
            Two buffer sets alternate by step parity, so step k's uploads
            overlap step k-1's launches and step k-1's downloads overlap step
            k's: a pipelined decode loop, every byte still crossing PCIe
            inside the timed region."""
            main = torch.cuda.current_stream(dev)
            c = state["cnt"]
            fork = torch.cuda.Event()
            fork.record(main)
            s_h2d.wait_event(fork)
            s_d2h.wait_event(fork)
            ran_ev, down_ev = {}, {}
            for k in range(args.steps):
                par = k & 1
                if k >= 2:
                    s_h2d.wait_event(ran_ev[k - 2])   # d_act[par] no longer read
                    main.wait_event(down_ev[k - 2])   # d_out[par] already downloaded
                with torch.cuda.stream(s_h2d):
                    d_act_all[par].copy_(h_act_all, non_blocking=True)
                    up = torch.cuda.Event()
                    up.record(s_h2d)
                main.wait_event(up)
                for n in batches:
                    launch(c, n, d_act[par][n].data_ptr(), d_out[par][n].data_ptr())
                    c += 1
                ran_ev[k] = torch.cuda.Event()
                ran_ev[k].record(main)
                s_d2h.wait_event(ran_ev[k])
                with torch.cuda.stream(s_d2h):
                    h_out_all.copy_(d_out_all[par], non_blocking=True)
                    down_ev[k] = torch.cuda.Event()
                    down_ev[k].record(s_d2h)
            j1, j2 = torch.cuda.Event(), torch.cuda.Event()
            j1.record(s_h2d)
            j2.record(s_d2h)
            main.wait_event(j1)
            main.wait_event(j2)

        g_e2e = capture(e2e_steps)
        e2e_ms = max_over_ranks(timed(g_e2e))
        h2d = tot_a * 2
        d2h = tot_c * 4
        e2e = {"value": round(world * nl * WEIGHT_BYTES / (e2e_ms * 1e-3) / 1e9, 1), "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(e2e_ms / args.steps, 4),
               "note": "per step: one H2D of the six batches' pinned host activations (copy stream) + the six "
                       "fpx_linear calls (C-ABI, compute stream) + one D2H of their fp32 outputs (second copy stream), "
                       "double-buffered so copies overlap the neighbouring steps' launches; replayed as one CUDA "
                       "graph; packed weights resident in HBM"}

    # ---- correctness spot check (untimed): last outputs vs a dequant+matmul
    W16 = fpx.dequantize(copies[0]).float()
    n_chk = batches[-1]
    ref = acts[n_chk].float() @ W16.t()
    got = fpx.gemm_packed(copies[0], acts[n_chk], split_k=splits[n_chk])
    rel = float(((got - ref).abs().amax(dim=1) / ref.abs().amax(dim=1)).max())
    del W16, ref

    hbm, hbm_src = peaks()
    traffic, traffic_src = ncu_traffic()
    value = world * nl * WEIGHT_BYTES / (total_ms * 1e-3) / 1e9
    # the timed region holds only fused-kernel launches (nl of them per rank):
    # its mean launch duration is the kernel's, measured live on its stream
    mean_launch_us = total_ms * 1e3 / nl
    achieved = WEIGHT_BYTES / (mean_launch_us * 1e-6) / 1e9
    res = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp6(e3m2) weights x fp16 activations -> fp32 (f16 MMA)",
        "data": "synthetic: N(0,0.02) weights quantized/packed on GPU, N(0,1) fp16 activations",
        "config": {"workload": "llama-65B FFN linear 8192x22016 FP6 e3m2, batch sweep 1/2/4/8/16/32 (one fused "
                               "linear per batch per step)", "M": M_ROWS, "K": K_COLS, "batches": batches,
                   "split_k": splits, "l2": "3 rotated packed-weight copies (405 MB > 126 MB L2)",
                   "parallelism": f"weak x{world} (independent output tiles per rank)"},
        "us_per_launch": {str(n): round(v, 2) for n, v in per_n.items()},
        "timing": "CUDA events around CUDA-graph replays of the K timed steps (host launch overhead excluded)",
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "traffic_source": f"{traffic_src} (N=16 launch, dram read+write bytes)" if traffic else None,
                     "peak_source": f"{hbm_src} MEASURED_PEAKS.json hbm_gbs" if hbm_src == "measured" else hbm_src,
                     "kernel": "fpx_linear_decode_kernel (mean device time per launch over the timed region: "
                               "K steps x the batch sweep, back to back)",
                     "us_per_launch": round(mean_launch_us, 2),
                     "algorithmic_bytes_per_launch": WEIGHT_BYTES},
        "gpu_launches": nl,  # one fused kernel per batch per step
        "clocks": clk.summary(),
        "e2e": e2e,
        "check": {"max_rel_err_vs_dequant_matmul": rel, "tol": 1e-2},
    }
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        res["cpu_baseline"] = cpu_baseline(codes_host, scales_host, batches, sample_batches=batches)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return res


# ------------------------------------------------------------ reference CPU
def _ref_setup(codes=None, scales=None):
    from oracle.oracle import REF_SO, Reference
    if not os.path.exists(REF_SO):
        return None, None
    R = Reference()
    if codes is None:
        rng = np.random.default_rng(1234)
        w = (rng.standard_normal((M_ROWS, K_COLS), dtype=np.float32) * np.float32(0.02))
        st, codes, scales = R.quantize(w, 3, 2)
        if st:
            raise RuntimeError(R.last_error())
    return R, R.prepare(codes, scales, 3, 2)


def cpu_baseline(codes, scales, batches, sample_batches):
    """Reference gemm_packed (unmodified, oracle/_ref) over the sweep once."""
    R, h = _ref_setup(codes, scales)
    if h is None:
        return {"value": None, "unit": "GB/s", "cores": os.cpu_count(), "kind": "reference",
                "sample": "oracle/_ref/libfpxref.so missing"}
    rng = np.random.default_rng(7)
    t = 0.0
    for n in sample_batches:
        b = rng.standard_normal((n, K_COLS)).astype(np.float16).view(np.uint16)
        t0 = time.perf_counter()
        h.gemm_packed(b)
        t += time.perf_counter() - t0
    return {"value": round(len(sample_batches) * WEIGHT_BYTES / t / 1e9, 4), "unit": "GB/s",
            "cores": int(os.environ.get("FPX_THREADS", os.cpu_count())), "kind": "reference",
            "sample": f"one pass of the batch sweep {list(sample_batches)} on the full 8192x22016 e3m2 weight "
                      f"({t:.1f} s, std::thread fan-out of the reference)", "seconds": round(t, 2)}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    batches = [int(x) for x in args.batches.split(",")]
    R, h = _ref_setup()
    if h is None:
        return {"impl": "reference", "unavailable": "oracle/_ref/libfpxref.so not built"}
    rng = np.random.default_rng(7)
    acts = {n: rng.standard_normal((n, K_COLS)).astype(np.float16).view(np.uint16) for n in batches}
    for _ in range(args.warmup):
        for n in batches:
            h.gemm_packed(acts[n])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for n in batches:
            h.gemm_packed(acts[n])
    dt = time.perf_counter() - t0
    value = args.steps * len(batches) * WEIGHT_BYTES / dt / 1e9
    cores = int(os.environ.get("FPX_THREADS", os.cpu_count()))
    return {"metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp6(e3m2) x fp16 -> fp32 (CPU soft-fp16 emulation)",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "llama-65B FFN linear 8192x22016 FP6 e3m2, batch sweep 1/2/4/8/16/32 (one "
                                   "gemm_packed per batch per step)", "M": M_ROWS, "K": K_COLS, "batches": batches},
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
                             "sample": f"full workload, {args.steps} steps"},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
