"""Pinned host <-> device copy bandwidth of this box (the floor of the e2e download).

    python tools/pcie_bw.py [MB]"""
import sys

import torch

mb = int(sys.argv[1]) if len(sys.argv) > 1 else 174
n = mb * 1000 * 1000
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for name, dst, src in (("D2H", host, dev), ("H2D", dev, host)):
    ts = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = sorted(ts)[len(ts) // 2]
    print(f"{name} {mb} MB pinned: {t:.3f} ms = {n / t / 1e6:.1f} GB/s")
