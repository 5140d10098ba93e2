"""hpl_load_factor at N (pinned host copy of the seeded system), printing the
pipelined start's timeline (HPL_PSTART_TRACE=1) and the phase stats."""
import sys
import time

import numpy as np

import paper_2304_10397_b200 as H

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
NB = int(sys.argv[2]) if len(sys.argv) > 2 else 512
with H.hpl_init(N, NB, 1, 1, 42) as ctx:
    host = H.hpl_get_local(ctx)
    H.hpl_pin_host(host, True)
    H.hpl_factor(ctx)
    H.hpl_solve(ctx, want_x=False)
    t = H.hpl_last_timing(ctx)
    print("plain factor+solve ms", t["factor_ms"] + t["solve_ms"], flush=True)
    t0 = time.perf_counter()
    H.hpl_load_factor(ctx, host)
    H.hpl_solve(ctx, want_x=False)
    print("load_factor wall s", time.perf_counter() - t0, flush=True)
    t = H.hpl_last_timing(ctx)
    print("device ms", t["factor_ms"] + t["solve_ms"], H.hpl_phase_stats(ctx), flush=True)
    H.hpl_pin_host(host, False)
