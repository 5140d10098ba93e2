"""One panel FACT (m x nb, default 8192 x 512: a tail panel of the C2 run,
where FACT is on the critical path) for ncu launch lists; prints the wall
time of a second call.
    python tools/fact_probe.py [m] [nb]"""
import sys
import time

import paper_2304_10397_b200 as H
from hpl_inputs import hpl_panel

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 512
P = hpl_panel(m, nb, seed=1)
H.hplk_panel_fact(P)
print("device ms per panel (hplk_panel_bench):", H.hplk_panel_bench(m, nb, 16, 0, 3))
