"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

Holds NONE of the method's arithmetic: only numpy RNG draws and library
factorizations (scipy/LAPACK) used to shape realistic test operands.  The
HPL matrix itself is generated on each side independently (oracle C vs the
CUDA generator, reading A6); this module never produces an
expected value.  Recipe: entries uniform on [-0.5, 0.5)
like the HPL generator; L/U operands are LAPACK factors of such matrices so
their conditioning matches what the trailing update sees (|L| <= 1).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg


def hpl_panel(m: int, nb: int, seed: int) -> np.ndarray:
    """A tall-skinny M x NB panel with HPL's value distribution."""
    return np.random.default_rng(seed).uniform(-0.5, 0.5, (m, nb))


def random_ipiv(rows: int, j0: int, jb: int, seed: int) -> np.ndarray:
    """Valid LAPACK pivots for block row j0: ipiv[k] in [j0+k, rows), with
    identity entries, swaps inside the block, and repeated targets below it."""
    rng = np.random.default_rng(seed)
    ipiv = np.empty(jb, dtype=np.int64)
    below = rng.integers(j0 + jb, rows, size=max(1, jb // 4)) if rows > j0 + jb else None
    for k in range(jb):
        r = rng.random()
        lo = j0 + k
        if r < 0.15 or lo == rows - 1:
            ipiv[k] = lo
        elif r < 0.35 and below is not None:
            ipiv[k] = below[rng.integers(0, len(below))]      # repeated targets
        else:
            ipiv[k] = rng.integers(lo, rows)
    return ipiv


def random_unit_lower(k: int, seed: int) -> np.ndarray:
    """Unit lower L (k x k) with |L| <= 1: the L factor LAPACK returns for a
    uniform random matrix (diagonal set to a junk value the solvers ignore)."""
    A = np.random.default_rng(seed).uniform(-0.5, 0.5, (k, k))
    _, L, _ = scipy.linalg.lu(A)
    return np.tril(L, -1) + np.eye(k) * 3.0


def upper_well_conditioned(n: int, seed: int) -> np.ndarray:
    """Upper triangular U factor of a uniform random matrix (LAPACK)."""
    A = np.random.default_rng(seed).uniform(-0.5, 0.5, (n, n))
    _, _, Uu = scipy.linalg.lu(A)
    return Uu


def _grid(rng, shape, lo, hi):
    """Uniform draws snapped to the 2^-53 grid (HPL's value set), in [lo, hi)."""
    return np.floor(rng.uniform(lo, hi, shape) * 2.0 ** 53) * 2.0 ** -53


def twin_panel(m: int, nb: int, seed: int, heavy: int | None = None) -> np.ndarray:
    """A panel built to make the pivot search see exact ties in every column
    (SPEC.md l.118 tie rule): `heavy` pairs of "twin" rows, each the exact
    negation of the other, with large entries, far apart (different CTAs /
    row chunks / process rows); every other row small.  Twins are updated
    symmetrically by elimination (the same operations on negated operands),
    so each column's maximum is shared by the two members of a pair until
    one is chosen; the rule must pick the smaller row index."""
    rng = np.random.default_rng(seed)
    heavy = heavy or min(nb, m // 4)
    P = _grid(rng, (m, nb), -0.01, 0.01)
    rows = rng.permutation(m)[: 2 * heavy]
    for t in range(heavy):
        a, b = int(rows[2 * t]), int(rows[2 * t + 1])
        v = _grid(rng, nb, 0.3, 0.5) * rng.choice([-1.0, 1.0], nb)
        P[a] = v
        P[b] = -v
    return P


def integer_panel(m: int, nb: int, seed: int, amax: int = 8) -> np.ndarray:
    """Small integers in [-amax, amax]: many equal |values| per column."""
    return np.random.default_rng(seed).integers(-amax, amax + 1, (m, nb)).astype(np.float64)


def twin_system(N: int, NB: int, P: int, seed: int) -> np.ndarray:
    """An N x (N+1) system [A | b] whose first panel's pivot search meets exact
    ties between rows on DIFFERENT process rows of a P-row grid (block row
    i // NB lives on process row (i // NB) % P): twin pairs as in twin_panel
    over the first NB columns, the rest of each row independent (A stays
    nonsingular).  The second member of a pair sits in the next block row,
    and every other pair is swapped so that the smaller index is sometimes
    on the higher process row."""
    rng = np.random.default_rng(seed)
    A = _grid(rng, (N, N + 1), -0.5, 0.5)
    w = min(NB, N)
    A[:, :w] = _grid(rng, (N, w), -0.01, 0.01)
    pairs = min(w, N // (2 * NB) * NB) if N >= 2 * NB else 0
    for t in range(pairs):
        blk = 2 * (t // NB)
        a = blk * NB + t % NB
        b = a + NB
        if b >= N:
            break
        if t % 2:
            a, b = b, a
        v = _grid(rng, w, 0.3, 0.5) * rng.choice([-1.0, 1.0], w)
        A[a, :w] = v
        A[b, :w] = -v
    return A


def local_block(Ab: np.ndarray, NB: int, P: int, Q: int, p: int, q: int) -> np.ndarray:
    """Process (p, q)'s local block of the global [A | b] (2D block-cyclic,
    NB x NB blocks, block (I, J) on (I mod P, J mod Q)) — index bookkeeping
    only, as hpl_load_local expects it (row-major, local rows x local cols)."""
    rows = [i for i in range(Ab.shape[0]) if (i // NB) % P == p]
    cols = [j for j in range(Ab.shape[1]) if (j // NB) % Q == q]
    return np.ascontiguousarray(Ab[np.ix_(rows, cols)])
