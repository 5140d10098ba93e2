"""Small end-to-end runs for compute-sanitizer (memcheck): every kernel of the
hot path on N=520 NB=64 (ragged), plus the kernel-level entry points."""
import numpy as np
import paper_2304_10397_b200 as H
from hpl_inputs import hpl_panel, random_ipiv, random_unit_lower
for (N, NB, la) in [(520, 64, 1), (256, 32, 0), (130, 16, 1)]:
    with H.hpl_init(N, NB, 1, 1, 7) as ctx:
        H.hpl_set_option(ctx, "lookahead", la)
        H.hpl_factor(ctx)
        x = H.hpl_solve(ctx)
        r = H.hpl_residual(ctx)
        assert r < 16, r
with H.hpl_init(300, 32, 1, 1, 3) as ctx:
    H.hpl_set_option(ctx, "split", 50)
    H.hpl_factor(ctx); H.hpl_solve(ctx); assert H.hpl_residual(ctx) < 16
H.hplk_panel_fact(hpl_panel(700, 48, 1))
H.hplk_trsm(random_unit_lower(64, 1), np.ones((64, 100)))
H.hplk_laswp(np.ones((300, 90)), 32, random_ipiv(300, 32, 32, 1), 3, 90)
H.hplk_dgemm_update(np.ones((130, 70)), np.ones((130, 33)), np.ones((33, 70)))
print("san_small ok")
