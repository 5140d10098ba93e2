import sys, numpy as np
import paper_2304_10397_b200 as H
import oracle
N, NB, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
opts = dict(a.split("=") for a in sys.argv[4:])
o = oracle.run(N, 42)
ok = 0
for rep in range(reps):
    with H.hpl_init(N, NB, 1, 1, 42) as ctx:
        for k, v in opts.items(): H.hpl_set_option(ctx, k, int(v))
        H.hpl_factor(ctx)
        ip = H.hpl_get_ipiv(ctx)
    ok += int(np.array_equal(ip, o["ipiv"]))
print(opts, "ok", ok, "of", reps, flush=True)
