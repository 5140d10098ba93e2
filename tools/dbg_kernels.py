import sys, numpy as np
import paper_2304_10397_b200 as H
from hpl_inputs import random_unit_lower
rng = np.random.default_rng(0)
for (m, n, k, cfg) in [(4096, 8000, 512, 2), (8000, 8000, 256, 2), (8000, 8000, 256, 0), (2000, 30000, 512, 2)]:
    A = rng.uniform(-1, 1, (m, k)); B = rng.uniform(-0.5, 0.5, (k, n)); C = rng.uniform(-0.5, 0.5, (m, n))
    got = H.hplk_dgemm_update(C, A, B, cfg=cfg)
    ref = C - A @ B
    d = np.abs(got - ref); bad = d > 1e-9
    print("gemm", m, n, k, cfg, "maxdiff", d.max(), "nbad", bad.sum(), flush=True)
for (k, n) in [(256, 7937), (512, 8000), (256, 30000)]:
    L = random_unit_lower(k, seed=k); Bm = rng.uniform(-0.5, 0.5, (k, n))
    got = H.hplk_trsm(L, Bm)
    Lf = np.tril(L, -1) + np.eye(k)
    ref = np.linalg.solve(Lf, Bm)
    d = np.abs(got - ref)
    bad = d > 1e-8 * np.abs(ref).max()
    r, c = np.nonzero(bad)
    print("trsm", k, n, "maxdiff", d.max(), "nbad", bad.sum(), "rows", np.unique(r)[:12], "cols", np.unique(c)[:6], flush=True)
