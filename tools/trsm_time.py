"""Time the DTRSM path (unit-lower inverse + a_lower DMMA GEMM) in isolation."""
import time, sys
import numpy as np
import paper_2304_10397_b200 as H
from hpl_inputs import random_unit_lower
k, n = int(sys.argv[1]), int(sys.argv[2])
L = random_unit_lower(k, 1); B = np.random.default_rng(0).uniform(-0.5, 0.5, (k, n))
H.hplk_trsm(L, B)
