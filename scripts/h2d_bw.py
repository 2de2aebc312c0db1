"""Pinned host->device bandwidth with the process bound to each NUMA node's CPUs."""
import os, sys, time
import torch
import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
words = pynvml.nvmlDeviceGetCpuAffinity(h, 64)
local = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
allc = sorted(os.sched_getaffinity(0))
print("cpus", len(allc), "gpu-local", len(local), local[:4], "...", flush=True)
other = [c for c in allc if c not in set(local)]


def bw(cpus, tag):
    os.sched_setaffinity(0, cpus)
    x = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    y = torch.empty_like(x, device="cuda")
    for _ in range(3):
        y.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        y.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(tag, "%.1f GB/s" % (10 * x.numel() / dt / 1e9), flush=True)


torch.cuda.init()
bw(local, "local")
if other:
    bw(other, "remote")
bw(allc, "all")
