"""DGEMM microbenchmark at HPL shapes (device-resident operands, CUDA events)."""
import json
import sys

import paper_2304_10397_b200 as H

shapes = [(32768, 32768, 512), (65536, 65536, 512), (130560, 130560, 512), (8192, 8192, 512),
          (4096, 4096, 512), (7936, 7936, 256)]
cfgs = [int(c) for c in sys.argv[1:]] or [2, 0, 1]
for (m, n, k) in shapes:
    for cfg in cfgs:
        ms = H.hplk_dgemm_bench(m, n, k, cfg=cfg, reps=3)
        tf = 2 * m * n * k / (min(ms) * 1e-3) / 1e12
        print(json.dumps(dict(m=m, n=n, k=k, cfg=cfg, ms=[round(v, 3) for v in ms], tflops=round(tf, 2))), flush=True)
