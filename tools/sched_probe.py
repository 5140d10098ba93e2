"""C2 schedule probe: the trailing DGEMM's live rate (flop / summed launch
events) and the step time under schedule options, one run each.

    python tools/sched_probe.py [N] [NB] [opt=v,opt=v ...]   (each arg = one run)"""
import json
import sys

import paper_2304_10397_b200 as H

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 512
runs = sys.argv[3:] or ["", "lookahead=0"]
for spec in runs:
    ctx = H.hpl_init(N, NB, 1, 1, 42)
    H.hpl_set_timing(ctx, True)
    opts = dict(kv.split("=") for kv in spec.split(",") if kv)
    for k, v in opts.items():
        H.hpl_set_option(ctx, k, int(v))
    H.hpl_factor(ctx)
    H.hpl_solve(ctx, want_x=False)
    t = H.hpl_last_timing(ctx)
    ps = H.hpl_phase_stats(ctx)
    ms = t["factor_ms"] + t["solve_ms"]
    fl = 2.0 / 3.0 * N ** 3 + 1.5 * N ** 2
    print(json.dumps(dict(opts=spec or "default", ms=round(ms, 1), tflops=round(fl / ms / 1e9, 3),
                          dgemm_live=round(t["dgemm_flop"] / t["dgemm_ms"] / 1e9, 3),
                          dgemm_ms=round(t["dgemm_ms"], 1), fact_ms=round(ps["fact_ms"], 1),
                          laswp_ms=round(ps["laswp_ms"], 1), trsm_ms=round(ps["trsm_ms"], 1))),
          flush=True)
    H.hpl_free(ctx)
