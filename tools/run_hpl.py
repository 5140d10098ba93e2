"""Time one HPL run (factor + solve) through the C ABI and print TFLOP/s + residual."""
import json
import sys
import time

import paper_2304_10397_b200 as H

N, NB = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
opts = dict(a.split("=") for a in sys.argv[4:])
t0 = time.time()
ctx = H.hpl_init(N, NB, 1, 1, 42)
for k, v in opts.items():
    H.hpl_set_option(ctx, k, int(v))
print("init s", round(time.time() - t0, 2), flush=True)
for r in range(reps):
    if r:
        H.hpl_regenerate(ctx)
    t0 = time.perf_counter()
    H.hpl_factor(ctx)
    t1 = time.perf_counter()
    x = H.hpl_solve(ctx)
    t2 = time.perf_counter()
    res = H.hpl_residual(ctx)
    fl = 2.0 / 3.0 * N ** 3 + 1.5 * N ** 2
    print(json.dumps(dict(N=N, NB=NB, factor_s=round(t1 - t0, 4), solve_s=round(t2 - t1, 4),
                          tflops=round(fl / (t2 - t0) / 1e12, 3), resid=res,
                          launches=H.hpl_launch_count(ctx))), flush=True)
H.hpl_free(ctx)
