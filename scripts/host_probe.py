"""Probe: host RAM, pinned H2D / D2H copy bandwidth (the host-DRAM tier's link)."""
import os
import subprocess
import time
import torch

print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout)
print(subprocess.run(["nproc"], capture_output=True, text=True).stdout)
n = 1 << 30
t0 = time.time()
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
print("pin 1 GiB s", time.time() - t0)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    print(name, "GB/s", 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9)
t0 = time.time()
big = torch.empty(16 << 30, dtype=torch.uint8, pin_memory=True)
print("pin 16 GiB s", time.time() - t0)
