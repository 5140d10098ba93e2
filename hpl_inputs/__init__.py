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
