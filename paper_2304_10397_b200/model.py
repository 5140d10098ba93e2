"""Timeline analysis and cost model for the HPL schedule (host-side, no GPU).

SURVEY.md §8(f) NEXT 2 and NEXT 4; PAPER.md l.70–84 (Fig. iteration, two
regimes), l.64 (hiding persistence), l.66 (split fraction)
(metrics-timeline: IterationTrace, overlap_fraction, predict_crossover,
tune_split).

Traces come from ``hpl_get_timeline`` (CUDA events inside libhpl): per
iteration j the ms spent in [FACT(j+1), look-ahead update, rest update, rest
RS/LASWP, rest DTRSM, rest DGEMM].  With depth-1 look-ahead the iteration's
critical path is max(rest, la + fact): the iteration is *hidden* when the
look-ahead chain (update of the next panel, FACT, LBCAST) fits under the
trailing update, *exposed* otherwise.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, List, Sequence

import numpy as np

QUANTUM = 0.05  # hidden <=> t_iter - t_engine <= 5 % of t_iter


@dataclass
class IterationTrace:
    j: int
    fact: float
    la: float
    rest: float
    rs: float
    trsm: float
    dgemm: float
    wall: float = 0.0     # replayed iteration time (0: derive from the phases)
    engine: float = 0.0   # replayed engine busy time (0: the rest phase)

    @property
    def t_iter(self) -> float:
        """Critical path of the iteration under depth-1 look-ahead."""
        return self.wall if self.wall > 0 else max(self.rest, self.la + self.fact)

    @property
    def t_engine(self) -> float:
        """Time the trailing-update engine is busy (the Fig. iteration 'GPU active')."""
        return self.engine if self.wall > 0 else self.rest


def traces_from_timeline(tl) -> List[IterationTrace]:
    tl = np.asarray(tl, dtype=np.float64)
    if tl.ndim == 2 and tl.shape[1] > 6:
        tl = tl[:, :6]  # extra columns (fact breakdown) are not phases of the model
    tl = tl.reshape(-1, 6)
    return [IterationTrace(j, *map(float, row)) for j, row in enumerate(tl)]


def regime(t: IterationTrace, quantum: float = QUANTUM) -> str:
    return "hidden" if t.t_iter - t.t_engine <= quantum * t.t_iter else "exposed"


def overlap_fraction(traces: Sequence[IterationTrace], quantum: float = QUANTUM) -> float:
    """Share of the run spent in hidden iterations (PAPER.md l.64 quotes ~75 %
    for rocHPL on one Frontier node): sum t_iter(hidden) / sum t_iter."""
    tot = sum(t.t_iter for t in traces)
    if tot <= 0:
        return 0.0
    return sum(t.t_iter for t in traces if regime(t, quantum) == "hidden") / tot


def crossover(traces: Sequence[IterationTrace], quantum: float = QUANTUM) -> int:
    """First iteration from which every later iteration is exposed (the
    Fig. iteration regime change); len(traces) if the run never crosses.  The
    last iteration has no next panel (no FACT, no look-ahead) and is neutral."""
    k = max(len(traces) - 1, 0)
    end = k
    while k > 0 and regime(traces[k - 1], quantum) == "exposed":
        k -= 1
    return k if k < end else len(traces)


# ----------------------------------------------------------------------------- model
@dataclass
class CostModel:
    """Per-phase costs (ms) as linear functions of the iteration's local sizes.

    rest  = c_gemm * 2 m n jb              (trailing DTRSM + DGEMM, flop-bound)
    la    = c_gemm * 2 m jb jb             (look-ahead update of jb columns)
    fact  = c_fact0 + c_fact1 * m          (latency floor + per-row work)
    rs    = c_rs * n jb                    (row-swap bytes)
    bcast = c_bcast * m jb                 (LBCAST bytes, 0 on one process column)
    """
    c_gemm: float
    c_fact0: float
    c_fact1: float
    c_rs: float = 0.0
    c_bcast: float = 0.0

    def phases(self, m: float, n: float, jb: float) -> dict:
        return dict(rest=self.c_gemm * 2 * m * n * jb + self.c_rs * n * jb,
                    la=self.c_gemm * 2 * m * jb * jb,
                    fact=self.c_fact0 + self.c_fact1 * m + self.c_bcast * m * jb,
                    rs=self.c_rs * n * jb)


def local_sizes(N: int, NB: int, P: int = 1, Q: int = 1):
    """(m_j, n_j, jb_j) per iteration: local rows at/below block row j and local
    trailing columns (incl. b) of one process, the average over the grid."""
    out = []
    for j in range(-(-N // NB)):
        j0 = j * NB
        jb = min(NB, N - j0)
        out.append(((N - j0) / P, (N + 1 - j0 - jb) / Q, jb))
    return out


def _features(N: int, NB: int, P: int, Q: int):
    """Per iteration j: (m, n, jb) of the trailing update and m' = rows of the
    NEXT panel (FACT(j+1) and the look-ahead update act on it; 0 at the end)."""
    sz = local_sizes(N, NB, P, Q)
    nxt = [sz[j + 1][0] if j + 1 < len(sz) else 0.0 for j in range(len(sz))]
    njb = [sz[j + 1][2] if j + 1 < len(sz) else 0 for j in range(len(sz))]
    return sz, nxt, njb


def predict(model: CostModel, N: int, NB: int, P: int = 1, Q: int = 1) -> List[IterationTrace]:
    tr = []
    sz, nxt, njb = _features(N, NB, P, Q)
    for j, (m, n, jb) in enumerate(sz):
        rest = model.c_gemm * 2 * m * n * jb + model.c_rs * n * jb
        la = model.c_gemm * 2 * nxt[j] * jb * njb[j]
        fact = (model.c_fact0 + model.c_fact1 * nxt[j] + model.c_bcast * nxt[j] * njb[j]
                if njb[j] else 0.0)
        rs = model.c_rs * n * jb
        tr.append(IterationTrace(j, fact, la, rest, rs, 0.0, rest - rs))
    return tr


def predict_crossover(model: CostModel, N: int, NB: int, P: int = 1, Q: int = 1,
                      quantum: float = QUANTUM) -> int:
    return crossover(predict(model, N, NB, P, Q), quantum)


def fit(traces: Sequence[IterationTrace], N: int, NB: int, P: int = 1, Q: int = 1) -> CostModel:
    """Least-squares fit of the model's coefficients to measured traces."""
    sz, nxt, njb = _features(N, NB, P, Q)
    k = len(traces)
    sz, nxt, njb = sz[:k], np.array(nxt[:k]), np.array(njb[:k])
    m = np.array([s[0] for s in sz]); n = np.array([s[1] for s in sz]); jb = np.array([s[2] for s in sz])
    rest = np.array([t.rest for t in traces]); fact = np.array([t.fact for t in traces])
    rs = np.array([t.rs for t in traces])
    gflop = 2 * m * n * jb
    ok = gflop > 0
    c_gemm = float(np.dot(gflop[ok], rest[ok] - rs[ok]) / np.dot(gflop[ok], gflop[ok]))
    has = njb > 0
    X = np.stack([np.ones_like(nxt[has]), nxt[has]], 1)
    c_fact0, c_fact1 = (float(v) for v in np.linalg.lstsq(X, fact[has], rcond=None)[0])
    byt = n * jb
    c_rs = float(np.dot(byt, rs) / max(np.dot(byt, byt), 1e-300))
    return CostModel(c_gemm=c_gemm, c_fact0=max(c_fact0, 0.0), c_fact1=max(c_fact1, 0.0),
                     c_rs=max(c_rs, 0.0))


# ----------------------------------------------------------------------------- split update
def split_iteration_hidden(model: CostModel, m: float, n1: float, n2: float, jb: float) -> bool:
    """Split update: UPDATE2 (right, n2 columns) must hide
    the look-ahead chain and RS1 (the left section's row swaps)."""
    upd2 = model.c_gemm * 2 * m * n2 * jb
    hidden = (model.c_gemm * 2 * m * jb * jb + model.c_fact0 + model.c_fact1 * m
              + model.c_bcast * m * jb + model.c_rs * n1 * jb)
    return upd2 >= hidden


def tune_split(model: CostModel, N: int, NB: int, P: int = 1, Q: int = 1) -> float:
    """Smallest right-section fraction n2/n (n2 a multiple of NB) whose UPDATE2
    hides the look-ahead chain and RS1 at iteration 0 (SPEC.md tune_split);
    1.0 if no fraction suffices."""
    m, n, jb = local_sizes(N, NB, P, Q)[0]
    for k in range(1, int(n // NB) + 1):
        n2 = k * NB
        if split_iteration_hidden(model, m, max(n - n2, 0.0), n2, jb):
            return n2 / n
    return 1.0


def hiding_persists(model: CostModel, N: int, NB: int, frac: float, P: int = 1,
                    Q: int = 1) -> bool:
    """with n2 fixed, UPDATE2 and the hidden phases both scale
    linearly in m (RS1 in n1, which shrinks), so if UPDATE2 hides them at the
    start it keeps hiding them while n1 > 0.  Checks that on the model."""
    sizes = local_sizes(N, NB, P, Q)
    n_local = sizes[0][1]
    n2 = max(NB, round(frac * n_local / NB) * NB)
    first = True
    for (m, n, jb) in sizes:
        n1 = n - n2
        if n1 <= 0:
            break
        ok = split_iteration_hidden(model, m, n1, n2, jb)
        if first and not ok:
            return True  # the premise does not hold: nothing to check
        first = False
        if not ok:
            return False
    return True


def summary(traces: Sequence[IterationTrace]) -> dict:
    return dict(iterations=len(traces), crossover=crossover(traces),
                overlap_fraction=overlap_fraction(traces),
                t_iter_ms=sum(t.t_iter for t in traces),
                exposed_ms=sum(max(0.0, t.la + t.fact - t.rest) for t in traces))


# ----------------------------------------------------------------------------- replay
@dataclass
class Replay:
    makespan: float
    traces: List[IterationTrace]


def _overlap(a0, a1, b0, b1):
    return max(0.0, min(a1, b1) - max(a0, b0))


def replay(model: CostModel, N: int, NB: int, P: int = 1, Q: int = 1, lookahead: bool = True,
           split: float = 0.0, alpha: float = 0.0) -> Replay:
    """Discrete-event replay of libhpl's stream schedule with model costs
    (SPEC.md MODEL mode).  Streams as in hpl_driver.cu:
    S_la (look-ahead update of panel j+1's columns, then FACT(j+1) after the
    trailing RS of iteration j), S_tr (trailing RS then DGEMM), and with
    ``split`` > 0 a third stream S_rs that runs RS_R(j), RS_L(j) while S_tr runs
    UPDATE_R(j), UPDATE_L(j) (the right section is a fixed
    NB-multiple share of the local columns, the schedule falls back once the
    left section is empty).  ``alpha`` stretches the trailing DGEMM by
    alpha × its overlap with a concurrent FACT (the SM-sharing slowdown).
    Per-iteration traces: t_iter = time between successive "trailing update
    of iteration j done and panel j+1 factored" marks, t_engine = DGEMM busy
    time, so the regime test of ``regime`` applies unchanged."""
    sz = local_sizes(N, NB, P, Q)
    J = len(sz)
    nxt = [sz[j + 1][0] if j + 1 < J else 0.0 for j in range(J)]
    njb = [sz[j + 1][2] if j + 1 < J else 0 for j in range(J)]
    fact_cost = [model.c_fact0 + model.c_fact1 * sz[0][0] + model.c_bcast * sz[0][0] * sz[0][2]]
    fact_cost += [(model.c_fact0 + model.c_fact1 * nxt[j] + model.c_bcast * nxt[j] * njb[j])
                  if njb[j] else 0.0 for j in range(J)]
    n2 = 0.0
    if split > 0:
        n2 = max(NB, round(split * sz[0][1] / NB) * NB) / 1.0
    fact_end = fact_cost[0]
    la_free = fact_end
    tr_free = 0.0
    rs_free = 0.0
    updR_end = updL_end = 0.0
    prev_mark = fact_end  # FACT(0) precedes iteration 0
    prev_rest_end = 0.0
    traces = []
    for j, (m, n, jb) in enumerate(sz):
        n_rest = max(n - njb[j], 0.0) if lookahead else n
        la = model.c_gemm * 2 * nxt[j] * jb * njb[j] if lookahead else 0.0
        fcost = fact_cost[j + 1]
        if not lookahead:
            rs_s = max(tr_free, fact_end)
            rs_e = rs_s + model.c_rs * n * jb
            up_e = rs_e + model.c_gemm * 2 * m * n * jb
            f_e = up_e + fcost
            tr_free = f_e
            mark = f_e
            traces.append(IterationTrace(j, fcost, 0.0, up_e - rs_s, rs_e - rs_s, 0.0, up_e - rs_e,
                                         wall=mark - prev_mark, engine=up_e - rs_s))
            fact_end = f_e
            prev_mark = mark
            continue
        # S_la: look-ahead update of panel j+1's columns (needs rest(j-1), FACT(j))
        la_s = max(la_free, fact_end, prev_rest_end)
        la_e = la_s + la
        n1 = n_rest - n2
        if split > 0 and n1 > 0:
            # S_rs: RS_R(j) then RS_L(j); S_tr: UPDATE_R(j) then UPDATE_L(j)
            rsR_s = max(rs_free, fact_end, updR_end)
            rsR_e = rsR_s + model.c_rs * n2 * jb
            rsL_s = max(rsR_e, updL_end)
            rsL_e = rsL_s + model.c_rs * n1 * jb
            rs_free = rsL_e
            f_s = max(la_e, rsR_e)
            f_e = f_s + fcost
            uR_s = max(tr_free, rsR_e)
            uR_d = model.c_gemm * 2 * m * n2 * jb
            uR_e = uR_s + uR_d
            uR_e += alpha * _overlap(uR_s, uR_e, f_s, f_e)
            uL_s = max(uR_e, rsL_e)
            uL_d = model.c_gemm * 2 * m * n1 * jb
            uL_e = uL_s + uL_d
            uL_e += alpha * _overlap(uL_s, uL_e, f_s, f_e)
            updR_end, updL_end = uR_e, uL_e
            rest_s, rs_e, rest_e = uR_s, rsL_e, uL_e
            dg = (uR_e - uR_s) + (uL_e - uL_s)
            rs_d = (rsR_e - rsR_s) + (rsL_e - rsL_s)
        else:
            rs_s = max(tr_free, fact_end, rs_free)
            rs_e = rs_s + model.c_rs * n_rest * jb
            f_s = max(la_e, rs_e)
            f_e = f_s + fcost
            up_d = model.c_gemm * 2 * m * n_rest * jb
            up_e = rs_e + up_d
            up_e += alpha * _overlap(rs_e, up_e, f_s, f_e)
            rest_s, rest_e = rs_s, up_e
            dg = up_e - rs_e
            rs_d = rs_e - rs_s
            updR_end = updL_end = rs_free = up_e
        tr_free = rest_e
        la_free = f_e
        mark = max(rest_e, f_e)
        # trace: la+fact on S_la vs the engine's busy time in this iteration
        traces.append(IterationTrace(j, f_e - f_s, la_e - la_s, dg + rs_d, rs_d, 0.0, dg,
                                     wall=max(mark - prev_mark, 1e-300), engine=dg + rs_d))
        prev_rest_end = rest_e
        fact_end = f_e
        prev_mark = mark
    return Replay(makespan=prev_mark, traces=traces)


def replay_regimes(rep: Replay, quantum: float = QUANTUM) -> List[str]:
    return [regime(t, quantum) for t in rep.traces]
