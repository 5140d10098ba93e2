"""Per-iteration phase timeline of one HPL run (CUDA events inside libhpl):
[fact, la_update, rest_update, rest_laswp, rest_trsm, rest_dgemm] ms per
iteration; prints a summary and writes the CSV (PAPER.md Fig. iteration analog)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_10397_b200 as H  # noqa: E402

N, NB = int(sys.argv[1]), int(sys.argv[2])
rest = sys.argv[3:]
opts = dict(a.split("=") for a in rest if "=" in a)
outs = [a for a in rest if "=" not in a]
out = outs[0] if outs else None
ctx = H.hpl_init(N, NB, 1, 1, 42)
for k, v in opts.items():
    H.hpl_set_option(ctx, k, int(v))
H.hpl_set_timing(ctx, True)
H.hpl_factor(ctx)                      # warm-up
H.hpl_regenerate(ctx)
H.hpl_factor(ctx)
H.hpl_solve(ctx, want_x=False)
t = H.hpl_last_timing(ctx)
tl = H.hpl_get_timeline(ctx)
fd = H.hpl_get_fact_detail(ctx)
r = H.hpl_residual(ctx)
H.hpl_free(ctx)
fact, la, rest, lsw, trsm, dg = tl.T
crit = np.maximum(rest, la + fact)
s = dict(N=N, NB=NB, opts=opts, factor_ms=t["factor_ms"], solve_ms=t["solve_ms"], resid=r,
         sum_rest=rest.sum(), sum_la=la.sum(), sum_fact=fact.sum(), sum_laswp=lsw.sum(),
         sum_trsm=trsm.sum(), sum_dgemm=dg.sum(), sum_crit=crit.sum(),
         exposed_iters=int(np.sum(la + fact > rest)),
         exposed_ms=float(np.sum(np.maximum(0, la + fact - rest))),
         dgemm_tflops=t["dgemm_flop"] / (t["dgemm_ms"] * 1e-3) / 1e12,
         sum_fact_wait=float(fd[:, 0].sum()), sum_fact_local=float(fd[:, 1].sum()),
         sum_lbcast_plan=float(fd[:, 2].sum()))
print(json.dumps({k: (v if k == "resid" else round(v, 3) if isinstance(v, float) else v)
                  for k, v in s.items()}))
if out:
    np.savetxt(out, tl, delimiter=",", header="fact,la_update,rest_update,rest_laswp,rest_trsm,rest_dgemm",
               fmt="%.4f")
