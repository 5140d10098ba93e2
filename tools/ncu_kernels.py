"""Representative single launches of the non-DGEMM hot-path kernels for ncu
(profiles/r02_ncu_*.md): run one mode per process under
    ncu --set full -k regex:<kernel> -c 1 -o <rep> python tools/ncu_kernels.py <mode>

modes (sizes of a mid-run C2 iteration, NB = 512):
  laswp  laswp_gs_kernel: 32768 x 32768 local block, jb = 512 rows swapped
  rs     rs_gather_peer / rs_scatter: the same over P = 2 emulated process rows
  trsm   the DTRSM as hpl_factor runs it: L11^{-1} (trsm_cols), then the
         a_lower ASSIGN DMMA GEMM on a 512 x 65536 U block row
  leaf   panel FACT of a 131072 x 512 panel with the hidden-FACT leaf grid
         (8 CTAs, grid leaf)
  solve  back solve of a 16384 x 16384 U (bs_partial, bs_diag_cluster)
"""
import sys

import numpy as np

import paper_2304_10397_b200 as H
from hpl_inputs import hpl_panel, random_ipiv, random_unit_lower

mode = sys.argv[1]
rng = np.random.default_rng(0)
if mode in ("laswp", "rs"):
    n = 32768
    A = rng.standard_normal((n, n))
    ipiv = random_ipiv(n, 4096, 512, seed=1)
    if mode == "laswp":
        H.hplk_laswp(A, 4096, ipiv, 0, n)
    else:
        H.hplk_rs_exchange(A, 512, 2, 4096, ipiv)
elif mode == "trsm":
    H.hplk_trsm(random_unit_lower(512, seed=3), rng.uniform(-0.5, 0.5, (512, 65536)))
elif mode == "leaf":
    H.hplk_panel_fact(hpl_panel(131072, 512, seed=4), nbmin=16, leaf_cluster=0, leaf_ctas=8)
elif mode == "solve":
    N = 16384
    U = np.triu(rng.uniform(-0.5, 0.5, (N, N))) + np.eye(N) * N ** 0.5
    H.hplk_back_solve(U, rng.uniform(-1, 1, N), NB=512)
else:
    raise SystemExit(f"unknown mode {mode}")
print("done", mode)
