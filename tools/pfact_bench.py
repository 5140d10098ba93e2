"""Device analog of PAPER.md Fig. pfact-mptest: panel FACT GFLOP/s of M x 512
panels (recursive right-looking, NDIV=2, base 16) vs M, for several leaf grid
widths (the device counterpart of the paper's CPU thread counts).
With --nbmin: the recursion base width NBMIN in {2, 4, 8, 16} instead;
with --variant: the leaf variant (right-looking, left-looking, Crout).  Flop count
M*NB^2 - NB^3/3.  Prints one JSON line per point."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_10397_b200 as H  # noqa: E402

NB = 512
nbmin_sweep = "--nbmin" in sys.argv
Ms = [int(v) for v in sys.argv[1:] if not v.startswith("--")] or \
    [1024, 2048, 4096, 8192, 16384, 32768, 65536, 131072]
if "--variant" in sys.argv:
    # leaf variant: right-looking / left-looking / Crout
    ctx = H.hpl_init(64, 16, 1, 1, 1)       # the knob is process-wide
    for M in Ms:
        for ctas in (8, 148):
            for var, name in ((0, "right"), (1, "left"), (2, "crout")):
                H.hpl_set_option(ctx, "leaf_variant", var)
                ms = H.hplk_panel_bench(M, NB, 16, ctas, reps=3)
                fl = M * NB ** 2 - NB ** 3 / 3
                print(json.dumps(dict(M=M, NB=NB, variant=name, leaf_ctas=ctas,
                                      ms=round(float(min(ms)), 3),
                                      gflops=round(fl / (min(ms) * 1e-3) / 1e9, 1))), flush=True)
    H.hpl_set_option(ctx, "leaf_variant", 0)
    H.hpl_free(ctx)
    sys.exit(0)
if nbmin_sweep:
    # recursion base width (PAPER.md l.34 uses 16 = LEAF_MAX here), all SMs and 8 CTAs
    for M in Ms:
        for ctas in (8, 148):
            for nbmin in (2, 4, 8, 16):
                ms = H.hplk_panel_bench(M, NB, nbmin, ctas, reps=3)
                fl = M * NB ** 2 - NB ** 3 / 3
                print(json.dumps(dict(M=M, NB=NB, nbmin=nbmin, leaf_ctas=ctas,
                                      ms=round(float(min(ms)), 3),
                                      gflops=round(fl / (min(ms) * 1e-3) / 1e9, 1))), flush=True)
    sys.exit(0)
for M in Ms:
    for ctas in (1, 2, 4, 8, 16, 32, 64, 148):
        ms = H.hplk_panel_bench(M, NB, 16, ctas, reps=3)
        fl = M * NB ** 2 - NB ** 3 / 3
        print(json.dumps(dict(M=M, NB=NB, leaf_ctas=ctas, ms=round(float(min(ms)), 3),
                              gflops=round(fl / (min(ms) * 1e-3) / 1e9, 1))), flush=True)
