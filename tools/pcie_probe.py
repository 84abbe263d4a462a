"""PCIe copy bandwidth from pinned host memory, with and without binding the
process to the GPU's NUMA-local CPUs (NVML affinity) before allocating the
pinned buffers (GPU box only)."""
import os
import time

import torch


def bw(nbytes, reps=20):
    dev = torch.device("cuda:0")
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    res = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    return res


def main():
    import pynvml
    pynvml.nvmlInit()
    hd = pynvml.nvmlDeviceGetHandleByIndex(0)
    ncpu = os.cpu_count()
    words = (ncpu + 63) // 64
    aff = pynvml.nvmlDeviceGetCpuAffinity(hd, words)
    local = [w * 64 + b for w, m in enumerate(aff) for b in range(64) if (m >> b) & 1]
    print(f"cpus {ncpu}, process affinity {len(os.sched_getaffinity(0))}, gpu-local cpus {len(local)} "
          f"({local[:4]}..{local[-2:]})")
    try:
        nodes = sorted(os.listdir("/sys/devices/system/node"))
        print("numa:", [n for n in nodes if n.startswith("node")])
    except OSError:
        pass
    for nb in (2_774_016, 64 << 20):
        print(f"unbound {nb/1e6:7.2f} MB", {k: round(v, 1) for k, v in bw(nb).items()})
    os.sched_setaffinity(0, local)
    for nb in (2_774_016, 64 << 20):
        print(f"bound   {nb/1e6:7.2f} MB", {k: round(v, 1) for k, v in bw(nb).items()})


if __name__ == "__main__":
    main()
