"""Per-configuration sweep of the fused FPx linear
next to cuBLAS FP16 on the same GPU -- a report, not the driver's bench line.

For every (shape, format, batch) it times, inside CUDA graphs of back-to-back
launches over enough rotated weight copies to exceed L2 (>= 3 x 126 MB):
  * fpx_linear through the C-ABI (default split, and the best of a split
    sweep when --sweep-splits is given);
  * torch.matmul with the fp16 weight (cuBLAS), the paper's baseline;
and prints one JSON line per case plus a markdown table (--md FILE).

  python bench_configs.py [--md profiles/rNN/configs.md] [--sweep-splits]
"""
import argparse
import ctypes as C
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_BYTES = 126 << 20

# (name, M, K, format (e, m), batches) -- SURVEY §8d
CONFIGS = [
    ("cfg1 4096x4096", 4096, 4096, (3, 2), [8]),
    ("cfg2 llama-65B FFN 8192x22016", 8192, 22016, (3, 2), [1, 2, 4, 8, 16, 32]),
    ("cfg2 transposed 22016x8192", 22016, 8192, (3, 2), [1, 16, 32]),
    ("cfg3 70B QKV 10240x8192", 10240, 8192, (3, 2), [16]),
    ("cfg3 70B O 8192x8192", 8192, 8192, (3, 2), [16]),
    ("cfg3 70B gate/up 28672x8192", 28672, 8192, (3, 2), [16]),
    ("cfg3 70B down 8192x28672", 8192, 28672, (3, 2), [16]),
    ("cfg4 e2m3 8192x22016", 8192, 22016, (2, 3), [1, 128]),
    ("cfg4 e2m2 8192x22016", 8192, 22016, (2, 2), [1, 128]),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--md", default=None)
    ap.add_argument("--sweep-splits", action="store_true")
    ap.add_argument("--launches", type=int, default=12)
    args = ap.parse_args()

    import torch

    import paper_2401_14112_b200 as fpx

    dev = torch.device("cuda:0")
    L = fpx._lib.load()
    peaks = {}
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        with open(pp) as f:
            peaks = json.load(f)
    hbm = float(peaks.get("hbm_gbs", 6527.5))

    def graph_time_us(fn, launches):
        torch.cuda.synchronize()
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(launches):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (2 * launches)

    rows_out = []
    for name, M, K, (e, m), batches in CONFIGS:
        fmt = fpx.FpxFormat(e, m)
        g = torch.Generator(device=dev)
        g.manual_seed(1)
        w = torch.randn(M, K, device=dev, generator=g) * 0.02
        p0 = fpx.pack(fpx.quantize_matrix(w, fmt))
        del w
        wbytes = M * K * fmt.total_bits / 8
        ncp = max(2, math.ceil(3 * L2_BYTES / wbytes))
        copies = [p0] + [fpx.PackedWeights(p0.format, p0.split, p0.rows, p0.cols, p0.orig_rows, p0.orig_cols,
                                           [s.clone() for s in p0.streams], p0.scales.clone()) for _ in range(ncp - 1)]
        ptrs = [(C.c_void_p * len(cp.streams))(*[s.data_ptr() for s in cp.streams]) for cp in copies]
        W16 = fpx.dequantize(p0)
        w16_copies = [W16] + [W16.clone() for _ in range(max(1, math.ceil(3 * L2_BYTES / (M * K * 2))) - 1)]
        for n in batches:
            act = (torch.randn(n, K, device=dev, generator=g)).half()
            out = torch.empty(n, M, device=dev)
            out16 = torch.empty(n, M, device=dev, dtype=torch.float16)
            split0 = fpx.default_split(M, K, n)
            cand = sorted({split0} | ({1, 2, 3, 4, 6, 8, 9, 12, 16} if args.sweep_splits else set()))
            res = {}
            for sp in cand:
                ws_n = int(L.fpx_linear_workspace_size(M, K, K, n, sp))
                ws = torch.zeros(max(ws_n, 16), dtype=torch.uint8, device=dev)

                def run(i, sp=sp, ws=ws):
                    cp = copies[i % ncp]
                    st = L.fpx_linear(ptrs[i % ncp], len(cp.streams), cp.scales.data_ptr(), M, K, e, m,
                                      act.data_ptr(), K, n, out.data_ptr(), M, sp, ws.data_ptr(), ws.numel(),
                                      torch.cuda.current_stream(dev).cuda_stream)  # the capture stream
                    if st:
                        raise RuntimeError(L.fpx_last_error().decode())

                res[sp] = graph_time_us(run, args.launches)
            ref = act.float() @ W16.float().t()
            err = float(((out - ref).abs().amax(dim=1) / ref.abs().amax(dim=1)).max())

            def cublas(i):
                torch.matmul(act, w16_copies[i % len(w16_copies)].t(), out=out16)

            t_cub = graph_time_us(cublas, args.launches)
            best_sp = min(res, key=res.get)
            t = res[split0]
            row = {"config": name, "M": M, "K": K, "format": fmt.name(), "n": n,
                   "weight_MB": round(wbytes / 1e6, 1), "split_default": split0, "us": round(t, 2),
                   "GBps": round(wbytes / t / 1e3, 1), "roofline_frac": round(wbytes / t / 1e3 / hbm, 3),
                   "TFLOPs": round(2.0 * M * K * n / t / 1e6, 1),
                   "split_best": best_sp, "us_best": round(res[best_sp], 2),
                   "cublas_fp16_us": round(t_cub, 2), "speedup_vs_cublas_fp16": round(t_cub / t, 2),
                   "max_rel_err": float(f"{err:.2e}"), "weight_copies": ncp}
            print(json.dumps(row), flush=True)
            rows_out.append(row)
        del copies, ptrs, w16_copies, W16
        torch.cuda.empty_cache()

    if args.md:
        hdr = ("| config | format | N | weight MB | µs | GB/s | roofline | TFLOP/s | split (best µs) | "
               "cuBLAS fp16 µs | speed-up |\n|---|---|---|---|---|---|---|---|---|---|---|\n")
        lines = [f"| {r['config']} | {r['format']} | {r['n']} | {r['weight_MB']} | {r['us']} | {r['GBps']} | "
                 f"{r['roofline_frac']} | {r['TFLOPs']} | {r['split_default']} ({r['split_best']}: {r['us_best']}) | "
                 f"{r['cublas_fp16_us']} | {r['speedup_vs_cublas_fp16']}x |" for r in rows_out]
        os.makedirs(os.path.dirname(os.path.abspath(args.md)), exist_ok=True)
        with open(args.md, "w") as f:
            f.write("# fpx_linear per configuration vs cuBLAS FP16 (bench_configs.py)\n\n"
                    f"HBM roofline denominator {hbm} GB/s (MEASURED_PEAKS.json). CUDA-graph replays of "
                    f"{args.launches} back-to-back launches over rotated weight copies (> 3x L2); fpx_linear "
                    "with its default split (and the best of the sweep when run with --sweep-splits).\n\n")
            f.write(hdr + "\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
