"""Host->device bandwidth of the local-matrix copy: one contiguous copy vs
column chunks (cudaMemcpy2DAsync, what hpl_load_factor issues), pinned.
    python tools/h2d_probe.py [rows] [cols] [chunks]"""
import sys
import time

import torch

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
chunks = [int(c) for c in sys.argv[3:]] or [1, 4, 16, 64]
h = torch.empty((rows, cols), dtype=torch.float64).pin_memory()
h.fill_(1.0)
d = torch.empty((rows, cols), dtype=torch.float64, device="cuda")
gb = rows * cols * 8 / 1e9
for nc in chunks:
    w = -(-cols // nc)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if nc == 1:
            d.copy_(h, non_blocking=True)
        else:
            for c0 in range(0, cols, w):
                d[:, c0:c0 + w].copy_(h[:, c0:c0 + w], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"chunks={nc:3d}: {gb / best:6.1f} GB/s ({best * 1e3:.1f} ms for {gb:.1f} GB)", flush=True)
