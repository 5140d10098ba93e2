import sys, numpy as np
import paper_2304_10397_b200 as H
from hpl_inputs import random_unit_lower
rng = np.random.default_rng(0)
k, n = int(sys.argv[1]), int(sys.argv[2])
L = random_unit_lower(k, seed=k); Bm = rng.uniform(-0.5, 0.5, (k, n))
Lf = np.tril(L, -1) + np.eye(k)
ref = np.linalg.solve(Lf, Bm)
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    got = H.hplk_trsm(L, Bm)
    d = np.abs(got - ref)
    bad = d > 1e-8 * np.abs(ref).max()
    r, c = np.nonzero(bad)
    print("trsm", k, n, "rep", rep, "nbad", bad.sum(), "rows", np.unique(r)[:8], "cols", np.unique(c)[:4], flush=True)
