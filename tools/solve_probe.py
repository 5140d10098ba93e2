"""Back-solve probe: hplk_back_solve (the look-ahead schedule of hpl_solve on
one rank) on a seeded upper-triangular U, for ncu launch lists.
    python tools/solve_probe.py [N] [NB] [reps]"""
import sys
import time

import numpy as np

import paper_2304_10397_b200 as H

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 512
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
rng = np.random.default_rng(0)
U = np.triu(rng.uniform(-0.5, 0.5, (N, N)))
U[np.arange(N), np.arange(N)] += np.sign(U[np.arange(N), np.arange(N)]) * N ** 0.5
y = rng.uniform(-1, 1, N)
for r in range(reps):
    t0 = time.perf_counter()
    x = H.hplk_back_solve(U, y, NB=NB)
    print(f"rep {r}: {1e3 * (time.perf_counter() - t0):.1f} ms (incl. H2D of U)", flush=True)
print("max|Ux-y|", float(np.max(np.abs(U @ x - y))))
