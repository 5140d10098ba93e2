"""Regime analysis of a measured per-iteration timeline:
hidden vs exposed iterations, crossover, overlap fraction,
the fitted cost model, its predicted crossover and the split fraction it suggests.

usage: python tools/regimes.py TIMELINE.csv N NB [P Q]
(the CSV is what tools/timeline.py writes)."""
import importlib.util
import json
import os
import sys

import numpy as np

_p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                  "paper_2304_10397_b200", "model.py")
_s = importlib.util.spec_from_file_location("hpl_model", _p)
M = importlib.util.module_from_spec(_s)
sys.modules["hpl_model"] = M
_s.loader.exec_module(M)

f, N, NB = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
P, Q = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (1, 1)
tr = M.traces_from_timeline(np.loadtxt(f, delimiter=",", skiprows=1))
c = M.fit(tr, N, NB, P, Q)
pred = M.predict(c, N, NB, P, Q)
out = dict(measured=M.summary(tr), regimes="".join("H" if M.regime(t) == "hidden" else "x" for t in tr),
           model=c.__dict__, predicted=M.summary(pred), tune_split=M.tune_split(c, N, NB, P, Q),
           replay_ms={"lookahead": M.replay(c, N, NB, P, Q).makespan,
                      "no_lookahead": M.replay(c, N, NB, P, Q, lookahead=False).makespan,
                      **{f"split_{f}": M.replay(c, N, NB, P, Q, split=f).makespan
                         for f in (0.1, 0.25, 0.5)}})
print(json.dumps(out, indent=1))
