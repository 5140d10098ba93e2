"""Replay the C2 run's trailing-DGEMM shapes in isolation (hplk_dgemm_bench,
one launch each, operands resident): the rate the rest updates would reach
with nothing beside them.  Compared with the live rate of the bench (FACT,
look-ahead update, LASWP and DTRSM share the SMs), it splits the DGEMM's loss
into shape effects (wave tails, small late updates) and interference.

    python tools/dgemm_sequence.py [N] [NB] [stride] [cfg]
"""
import json
import sys

import numpy as np

import paper_2304_10397_b200 as H

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 512
stride = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = int(sys.argv[4]) if len(sys.argv) > 4 else -1
nblk = -(-N // NB)
flop = t = 0.0
rows = []
for j in range(0, nblk - 1, stride):
    m = N - (j + 1) * NB                       # rows below block row j
    n = (N + 1) - (j + 2) * NB                 # rest columns (panel j+1 is the look-ahead)
    if m <= 0 or n <= 0:
        continue
    ms = float(np.min(H.hplk_dgemm_bench(m, n, NB, cfg, 2)))
    f = 2.0 * m * n * NB
    flop += f * stride
    t += ms * 1e-3 * stride
    rows.append((j, m, n, ms, f / (ms * 1e-3) / 1e12))
print(json.dumps(dict(N=N, NB=NB, stride=stride, cfg=cfg, tflops=flop / t / 1e12, seconds=t,
                      first=rows[0], mid=rows[len(rows) // 2], last=rows[-1])))
