"""Is host DRAM the cap of the hybrid e2e path?  Host read roof (scripts/host_read_bw.c, T pinned threads) alone, a pinned H2D
DMA loop alone, and both at once.  If CPU + DMA together stay near the CPU-only figure, DRAM (or the VM's share of it) is the cap."""
import os
import subprocess
import sys
import threading
import time

import torch

here = os.path.dirname(os.path.abspath(__file__))
exe = "/tmp/hrbw"
subprocess.run(["gcc", "-O3", "-march=native", "-pthread", os.path.join(here, "host_read_bw.c"), "-o", exe], check=True)
torch.cuda.set_device(0)
src = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True).fill_(1)
dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
stop = False
rate = [0.0]


def dma_loop():
    s = torch.cuda.Stream()
    n = 0
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        while not stop:
            dst.copy_(src, non_blocking=True)
            s.synchronize()
            n += 1
    rate[0] = n * src.numel() / (time.perf_counter() - t0) / 1e9


for threads in (15, 16):
    out = subprocess.run([exe, str(threads)], capture_output=True, text=True).stdout.strip()
    print("CPU alone :", out, flush=True)
    stop = False
    th = threading.Thread(target=dma_loop)
    th.start()
    time.sleep(0.5)
    out = subprocess.run([exe, str(threads)], capture_output=True, text=True).stdout.strip()
    stop = True
    th.join()
    print(f"CPU + DMA : {out}   | DMA meanwhile {rate[0]:.1f} GB/s (incl. the CPU test's first-touch phase)", flush=True)
stop = False
th = threading.Thread(target=dma_loop)
th.start()
time.sleep(3)
stop = True
th.join()
print(f"DMA alone : {rate[0]:.1f} GB/s")
