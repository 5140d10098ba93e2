"""CPU tests of the timeline analysis / cost model (paper_2304_10397_b200/model.py),
pinned to closed forms and the properties SPEC.md l.467–470 states."""
import importlib.util
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location(
    "hpl_model", os.path.join(ROOT, "paper_2304_10397_b200", "model.py"))
M = importlib.util.module_from_spec(_spec)
sys.modules["hpl_model"] = M
_spec.loader.exec_module(M)


def _tr(rows):
    return M.traces_from_timeline(np.array(rows, dtype=float))


def test_overlap_fraction_extremes():
    # all hidden -> 1.0, none hidden -> 0.0
    hidden = _tr([[1, 1, 10, 0, 0, 10]] * 5)
    exposed = _tr([[10, 1, 2, 0, 0, 2]] * 5)
    assert M.overlap_fraction(hidden) == 1.0
    assert M.overlap_fraction(exposed) == 0.0
    assert M.crossover(hidden) == 5 and M.crossover(exposed) == 0


def test_two_regime_crossover_and_fraction():
    # rest shrinks quadratically, fact linearly: one hidden->exposed transition
    rows = []
    for j in range(100):
        s = 1 - j / 100
        rows.append([5 * s + 1, 0.1, 100 * s * s, 0, 0, 100 * s * s])
    tr = _tr(rows)
    k = M.crossover(tr)
    regimes = [M.regime(t) for t in tr]
    assert all(r == "hidden" for r in regimes[:k]) and all(r == "exposed" for r in regimes[k:])
    # exact crossover of 100 s^2 vs 5 s + 1.1 (quantum 5 %): first s where exposed
    s = 1 - np.arange(100) / 100
    exposed = (np.maximum(100 * s * s, 5 * s + 1.1) - 100 * s * s) > 0.05 * np.maximum(100 * s * s, 5 * s + 1.1)
    assert k == int(np.argmax(exposed))
    assert 0.0 < M.overlap_fraction(tr) < 1.0


def test_zero_fact_cost_never_crosses():
    # zero communication / FACT cost -> crossover at the end
    m = M.CostModel(c_gemm=1e-9, c_fact0=0.0, c_fact1=0.0)
    assert M.predict_crossover(m, 8192, 256) >= len(M.local_sizes(8192, 256)) - 1


def test_dominant_fact_crosses_at_zero():
    m = M.CostModel(c_gemm=1e-12, c_fact0=1e6, c_fact1=0.0)
    assert M.predict_crossover(m, 8192, 256) == 0


def test_crossover_monotone_in_fact_cost():
    # raising a hidden-phase coefficient never delays the crossover
    ks = [M.predict_crossover(M.CostModel(3e-11, f, 1e-5), 131072, 512) for f in (0.5, 2, 8, 32)]
    assert all(a >= b for a, b in zip(ks, ks[1:]))


def test_fit_recovers_coefficients():
    true = M.CostModel(c_gemm=2.8e-11, c_fact0=4.5, c_fact1=2.0e-4, c_rs=3e-6)
    tr = M.predict(true, 65536, 512, 2, 2)
    got = M.fit(tr, 65536, 512, 2, 2)
    assert got.c_gemm == pytest.approx(true.c_gemm, rel=1e-9)
    assert got.c_fact0 == pytest.approx(true.c_fact0, rel=1e-6)
    assert got.c_fact1 == pytest.approx(true.c_fact1, rel=1e-6)
    assert got.c_rs == pytest.approx(true.c_rs, rel=1e-6)


def test_tune_split_properties():
    # zero hidden-phase cost -> the minimal fraction NB / n (SPEC tune_split example)
    m0 = M.CostModel(c_gemm=1e-11, c_fact0=0.0, c_fact1=0.0)
    n = M.local_sizes(65536, 512, 2, 2)[0][1]
    assert M.tune_split(m0, 65536, 512, 2, 2) == pytest.approx(512 / n)
    # a heavier FACT needs a larger right section
    a = M.tune_split(M.CostModel(1e-11, 50.0, 1e-4, c_rs=1e-6), 65536, 512, 2, 2)
    b = M.tune_split(M.CostModel(1e-11, 200.0, 1e-4, c_rs=1e-6), 65536, 512, 2, 2)
    assert a <= b <= 1.0


def test_hiding_persistence():
    # hidden at the start => hidden while n1 > 0 (linear-in-m costs)
    for c in [M.CostModel(1e-11, 0.0, 1e-4, c_rs=1e-6, c_bcast=1e-7),
              M.CostModel(3e-11, 0.0, 5e-4, c_rs=5e-6)]:
        f = M.tune_split(c, 131072, 512, 2, 2)
        if f < 1.0:
            assert M.hiding_persists(c, 131072, 512, f, 2, 2)


# ---- discrete-event replay (SPEC.md MODEL mode)
def _rand_models(k, seed=0):
    rng = np.random.default_rng(seed)
    return [M.CostModel(c_gemm=rng.uniform(1e-11, 4e-11), c_fact0=rng.uniform(0, 20),
                        c_fact1=rng.uniform(0, 5e-4), c_rs=rng.uniform(0, 2e-8))
            for _ in range(k)]


def test_replay_lookahead_matches_recurrence():
    # independent statement of the depth-1 look-ahead critical path (rs = 0):
    # R_j = max(R_{j-1}, F_j) + u_j ;  F_{j+1} = max(F_j, R_{j-1}) + la_j + f_{j+1}
    c = M.CostModel(c_gemm=3e-11, c_fact0=7.0, c_fact1=2e-4)
    N, NB = 32768, 512
    s = M.local_sizes(N, NB)
    J = len(s)
    f = [c.c_fact0 + c.c_fact1 * s[0][0]] + [c.c_fact0 + c.c_fact1 * s[j + 1][0] if j + 1 < J else 0.0
                                            for j in range(J)]
    R_prev, F = 0.0, f[0]
    for j, (m, n, jb) in enumerate(s):
        nj = s[j + 1][2] if j + 1 < J else 0
        mj = s[j + 1][0] if j + 1 < J else 0.0
        u = c.c_gemm * 2 * m * max(n - nj, 0) * jb
        la = c.c_gemm * 2 * mj * jb * nj
        R = max(R_prev, F) + u
        F = max(F, R_prev) + la + f[j + 1]
        R_prev = R
    assert M.replay(c, N, NB).makespan == pytest.approx(max(R_prev, F), rel=1e-12)


def test_replay_no_lookahead_closed_form():
    c = M.CostModel(c_gemm=3e-11, c_fact0=7.0, c_fact1=2e-4, c_rs=1e-8)
    N, NB = 32768, 512
    s = M.local_sizes(N, NB)
    tot = c.c_fact0 + c.c_fact1 * N
    for j, (m, n, jb) in enumerate(s):
        tot += c.c_rs * n * jb + c.c_gemm * 2 * m * n * jb
        if j + 1 < len(s):
            tot += c.c_fact0 + c.c_fact1 * s[j + 1][0]
    assert M.replay(c, N, NB, lookahead=False).makespan == pytest.approx(tot, rel=1e-12)


def test_replay_lookahead_never_slower_and_crossover_agrees():
    # SPEC.md: predicted crossover within +-2 iterations of the simulated flip
    for c in _rand_models(5):
        la = M.replay(c, 65536, 512)
        assert la.makespan <= M.replay(c, 65536, 512, lookahead=False).makespan * (1 + 1e-12)
        assert abs(M.crossover(la.traces) - M.predict_crossover(c, 65536, 512)) <= 2
        reg = M.replay_regimes(la)[:-1]
        flips = sum(1 for a, b in zip(reg, reg[1:]) if a != b)
        assert flips <= 1 and (not reg or reg[0] == "hidden" or "hidden" not in reg)


def test_replay_split_degenerates_and_persists():
    c = M.CostModel(c_gemm=1e-11, c_fact0=0.0, c_fact1=1e-4, c_rs=5e-6)
    N, NB = 65536, 512
    # right section covering all columns -> the unsplit schedule
    assert M.replay(c, N, NB, split=1.0).makespan == pytest.approx(M.replay(c, N, NB).makespan,
                                                                    rel=1e-12)
    # hidden at iteration 0 -> hidden while the left section is non-empty
    f = M.tune_split(c, N, NB)
    assert f < 1.0
    rep = M.replay(c, N, NB, split=f)
    n2 = max(NB, round(f * M.local_sizes(N, NB)[0][1] / NB) * NB)
    for t, (m, n, jb) in zip(rep.traces, M.local_sizes(N, NB)):
        if n - jb - n2 > 0:
            assert M.regime(t) == "hidden", t.j
