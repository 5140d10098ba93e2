import json, sys
import paper_2304_10397_b200 as H
cfgs = [int(c) for c in sys.argv[1:]] or [2, 4]
for m in (65536, 32768, 8192):
    for cfg in cfgs:
        ms = H.hplk_dgemm_bench(m, m, 512, cfg=cfg, reps=3)
        print(json.dumps(dict(m=m, cfg=cfg, ms=round(min(ms), 3), tflops=round(2 * m * m * 512 / (min(ms) * 1e-3) / 1e12, 2))), flush=True)
