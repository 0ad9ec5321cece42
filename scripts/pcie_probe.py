"""PCIe ceiling for the e2e leg: pinned H2D / D2H of one c2 vector, alone and
overlapped; with the process bound to the GPU's NUMA-local CPUs (NVML CPU
affinity) before the pinned buffers are allocated, and without."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_18020_b200._device import bind_gpu_local_cpus  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "local"
if mode == "local":
    print("bound to", bind_gpu_local_cpus(0))
n = 686433
if mode == "tf":  # cudaHostAlloc-backed (paper_2604_18020_b200._device.pinned_empty)
    from paper_2604_18020_b200._device import pinned_empty

    h_in = pinned_empty(n, torch.float32)
    h_in.copy_(torch.randn(n))
    h_out = pinned_empty(n, torch.float32)
else:
    h_in = torch.randn(n).pin_memory()
    h_out = torch.empty(n).pin_memory()
d_in = torch.empty(n, device="cuda")
d_out = torch.randn(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
# the PCIe link downshifts while idle: ~100 ms of traffic first, then measure
for _ in range(1000):
    d_in.copy_(h_in, non_blocking=True)
    h_out.copy_(d_out, non_blocking=True)
torch.cuda.synchronize()
for label, both in (("h2d", 0), ("d2h", 1), ("both", 2)):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 200
    e0.record()
    for _ in range(reps):
        if both in (0, 2):
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if both in (1, 2):
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"[{mode}] {label}: {us:.1f} us per 2.75 MB vector -> {n * 4 / us / 1e3:.1f} GB/s per direction")
