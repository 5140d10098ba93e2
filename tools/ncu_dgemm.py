"""Two launches of the trailing-update DGEMM (warm-up + measured) at an HPL
shape, for `ncu --set full -k regex:dgemm -s 1 -c 1`."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2304_10397_b200 as H  # noqa: E402
m = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
ms = H.hplk_dgemm_bench(m, m, 512, cfg=-1, reps=1)
print("ms", ms, "TF", 2 * m * m * 512 / (ms[0] * 1e-3) / 1e12)
