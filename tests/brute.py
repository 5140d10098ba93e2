"""Exact-arithmetic brute force used to PIN the oracle (tests only).

Nothing here is the oracle's formulation: pivots are chosen in exact rational
arithmetic, determinants come from the Leibniz permutation sum, and bounds are
the textbook backward-error bounds (Higham, "Accuracy and Stability of
Numerical Algorithms", 2nd ed., Thm 9.3 for LU, §3.5 for inner products).
"""
from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np


def to_frac(A):
    A = np.asarray(A, dtype=np.float64)
    if A.ndim == 1:
        return [Fraction(float(v)) for v in A]
    return [[Fraction(float(v)) for v in row] for row in A]


def exact_gepp(A):
    """GEPP in exact rationals on the (exactly representable) double input.
    Returns (L, U, perm_rows, ipiv) with P A = L U exactly, ipiv LAPACK-style."""
    n = len(A)
    m = len(A[0])
    W = [row[:] for row in A]
    ipiv = []
    L = [[Fraction(0)] * min(n, m) for _ in range(n)]
    for k in range(min(n, m)):
        p = max(range(k, n), key=lambda i: (abs(W[i][k]), -i))
        ipiv.append(p)
        if W[p][k] == 0:
            return None, None, None, ipiv  # singular at column k
        W[k], W[p] = W[p], W[k]
        L[k], L[p] = L[p], L[k]
        for i in range(k + 1, n):
            f = W[i][k] / W[k][k]
            L[i][k] = f
            for c in range(k, m):
                W[i][c] -= f * W[k][c]
    for k in range(min(n, m)):
        L[k][k] = Fraction(1)
    U = [[W[i][c] if c >= i else Fraction(0) for c in range(m)] for i in range(min(n, m))]
    return L, U, W, ipiv


def det_leibniz(A):
    """Determinant by the permutation (Leibniz) sum — exact, O(n! n)."""
    n = len(A)
    total = Fraction(0)
    for perm in itertools.permutations(range(n)):
        # sign by counting inversions
        inv = sum(1 for i in range(n) for j in range(i + 1, n) if perm[i] > perm[j])
        prod = Fraction(1)
        for i in range(n):
            prod *= A[i][perm[i]]
            if prod == 0:
                break
        total += -prod if inv % 2 else prod
    return total


def cramer(A, b):
    """x_i = det(A_i) / det(A) with A_i = A with column i replaced by b."""
    n = len(A)
    d = det_leibniz(A)
    xs = []
    for i in range(n):
        Ai = [row[:] for row in A]
        for r in range(n):
            Ai[r][i] = b[r]
        xs.append(det_leibniz(Ai) / d)
    return xs


def perm_from_ipiv(ipiv, n):
    """Row order produced by applying swaps k <-> ipiv[k] in sequence."""
    order = list(range(n))
    for k, p in enumerate(ipiv):
        order[k], order[p] = order[p], order[k]
    return order


def gamma(n: int, u: float = 2.0 ** -53) -> float:
    return n * u / (1 - n * u)
