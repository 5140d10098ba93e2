"""Per-tile overhead probe of the trailing DGEMM: the same m x n at k = 512,
1024, 2048 (one CTA tile's mainloop grows with k, its prologue/epilogue do
not), under the default epilogue and the options gemm_red / gemm_tpc.

    python tools/gemm_overhead.py [m]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_10397_b200 as H  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
peak = H.hplk_dmma_peak()
print(json.dumps(dict(dmma_peak=peak)), flush=True)
ctx = H.hpl_init(1024, 64, 1, 1, 1)   # only to reach the global kernel options
for opts in ({}, {"gemm_red": 1}, {"gemm_tpc": 2}, {"gemm_tpc": 4}):
    for k, v in {"gemm_red": 0, "gemm_tpc": 1, **opts}.items():
        H.hpl_set_option(ctx, k, v)
    for k in (512, 1024, 2048):
        ms = min(H.hplk_dgemm_bench(m, m, k, cfg=2, reps=5))
        tf = 2 * m * m * k / (ms * 1e-3) / 1e12
        print(json.dumps(dict(opts=opts, m=m, k=k, ms=round(ms, 3), tflops=round(tf, 3),
                              frac_dmma=round(tf / peak, 4))), flush=True)
H.hpl_free(ctx)
