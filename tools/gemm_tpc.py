import json, sys
import paper_2304_10397_b200 as H
for m in (65536, 32768, 16384):
    for tpc in (1, 2, 4, 8):
        ms = H.hplk_dgemm_bench(m, m, 512, cfg=100 * tpc + 2, reps=3)
        print(json.dumps(dict(m=m, tpc=tpc, ms=round(min(ms), 3), tflops=round(2 * m * m * 512 / (min(ms) * 1e-3) / 1e12, 2))), flush=True)
