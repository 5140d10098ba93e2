"""Pins for the CPU oracle (-m "not gpu").  Each test ties an oracle function
to something other than itself: a published test vector, exact-rational
brute force, a closed form, a library routine (LAPACK via scipy), or an
invariant stated in SPEC.md / the LU error analysis.  See DESIGN.md §Parity.
"""
from __future__ import annotations

import os
import subprocess
import sys
from fractions import Fraction

import numpy as np
import pytest
import scipy.linalg

import oracle
from tests import brute

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
U = 2.0 ** -53


# ---------------------------------------------------------------- O1 generator
def test_splitmix64_public_vector():
    """SplitMix64 seed-0 outputs (tests/golden/splitmix64_seed0.txt, cited)."""
    rows = [l.split() for l in open(os.path.join(ROOT, "tests/golden/splitmix64_seed0.txt"))
            if l.strip() and not l.startswith("#")]
    for k, hexv in rows:
        assert oracle.splitmix64(0, int(k)) == int(hexv, 16)


def test_generator_range_grid_and_stats():
    """entries in [-0.5, 0.5], 64x64 sample mean in (-0.05, 0.05);
    values lie on the 2^-53 grid (reading A6: exact 53-bit map)."""
    A, b = oracle.generate(7, 64)
    allv = np.concatenate([A.ravel(), b])
    assert allv.min() >= -0.5 and allv.max() < 0.5
    assert abs(A.mean()) < 0.05
    scaled = allv * 2.0 ** 53
    assert np.all(scaled == np.round(scaled))
    # top-53-bit map: value*2^53 + 2^52 == splitmix >> 11 for a few entries
    N = 64
    for (i, j) in [(0, 0), (5, 17), (63, 63), (3, N)]:
        z = oracle.splitmix64(7, j * N + i)
        assert oracle.gen_entry(7, N, i, j) * 2.0 ** 53 + 2.0 ** 52 == float(z >> 11)


def test_generator_pure_function_no_alias():
    """value is a pure function of (seed, i, j) — identical
    whether produced by the full fill or by single-entry calls; b (column N)
    does not alias A[i+1][0] (reading A6 fixes SPEC's i*N+j aliasing)."""
    N = 32
    A, b = oracle.generate(42, N)
    for (i, j) in [(0, 0), (31, 0), (7, 9), (0, 31)]:
        assert A[i, j] == oracle.gen_entry(42, N, i, j)
    for i in range(N - 1):
        assert b[i] != A[i + 1, 0]
    assert len(np.unique(np.concatenate([A.ravel(), b]))) == N * N + N


# ---------------------------------------------------------------- O2 GEPP
@pytest.mark.parametrize("n,seed", [(2, 1), (3, 2), (5, 3), (8, 4), (8, 5)])
def test_getrf_exact_rational_brute_force(n, seed):
    """Pivots identical to exact-rational GEPP on the same doubles; factors
    within the LU backward-error bound |PA - LU| <= gamma_n |L||U| (Higham Thm 9.3)."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-0.5, 0.5, (n, n))
    LU, ipiv, info = oracle.getrf(A)
    assert info == -1
    Lx, Ux, _, ipx = brute.exact_gepp(brute.to_frac(A))
    assert list(ipiv) == ipx
    L = np.tril(LU, -1) + np.eye(n)
    Uf = np.triu(LU)
    # factors vs exact factors (well-conditioned tiny cases)
    Lxe = np.array([[float(v) for v in r] for r in Lx])
    Uxe = np.array([[float(v) for v in r] for r in Ux])
    assert np.allclose(L, Lxe, rtol=0, atol=1e-13)
    assert np.allclose(Uf, Uxe, rtol=0, atol=1e-13)
    order = brute.perm_from_ipiv(ipiv, n)
    PA = A[order]
    bound = brute.gamma(n) * (np.abs(L) @ np.abs(Uf))
    assert np.all(np.abs(PA - L @ Uf) <= bound + 1e-300)


@pytest.mark.parametrize("n,seed", [(3, 11), (5, 12), (7, 13)])
def test_solve_vs_cramer(n, seed):
    """x from the oracle's getrf+getrs vs Cramer's rule in exact rationals."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-0.5, 0.5, (n, n))
    b = rng.uniform(-0.5, 0.5, n)
    LU, ipiv, info = oracle.getrf(A)
    x = oracle.getrs(LU, ipiv, b)
    xc = brute.cramer(brute.to_frac(A), brute.to_frac(b))
    xe = np.array([float(v) for v in xc])
    cond = np.linalg.cond(A, np.inf)
    assert np.max(np.abs(x - xe)) / np.max(np.abs(xe)) <= 64 * n * U * cond


def test_getrf_special_cases():
    # NB=1 panel [[0],[3]] -> swap, L=[1,0]^T, U=[3], ipiv=[1]
    LU, ipiv, info = oracle.getrf(np.array([[0.0], [3.0]]))
    assert info == -1 and list(ipiv) == [1] and LU[0, 0] == 3.0 and LU[1, 0] == 0.0
    # identity: L=U=I, ipiv = id
    LU, ipiv, info = oracle.getrf(np.eye(4))
    assert list(ipiv) == [0, 1, 2, 3] and np.array_equal(LU, np.eye(4))
    # permutation matrix: x = P^T b exactly
    perm = [2, 0, 3, 1]
    Pm = np.eye(4)[perm]
    b = np.array([1.0, -2.0, 3.5, 0.25])
    LU, ipiv, info = oracle.getrf(Pm)
    x = oracle.getrs(LU, ipiv, b)
    assert np.array_equal(x, Pm.T @ b)
    # exact zero column -> singular at that column (reading A3)
    A = np.array([[1.0, 2.0, 3.0], [2.0, 4.0, 1.0], [3.0, 6.0, 2.0]])  # col1 = 2*col0
    _, _, info = oracle.getrf(A)
    assert info == 1
    # tie rule: |a| ties -> smallest row
    _, ipiv, _ = oracle.getrf(np.array([[1.0, 0.0], [-2.0, 1.0], [2.0, 5.0]]))
    assert ipiv[0] == 1


@pytest.mark.parametrize("N,seed", [(256, 42), (512, 1), (1000, 7)])
def test_getrf_matches_lapack(N, seed):
    """Library pin: LAPACK dgetrf (scipy/OpenBLAS) chooses identical pivots on the
    seeded HPL matrix, and x agrees with dgesv."""
    A, b = oracle.generate(seed, N)
    LU, ipiv, info = oracle.getrf(A)
    lu_l, piv_l = scipy.linalg.lu_factor(A)
    assert np.array_equal(ipiv, piv_l.astype(np.int64))
    x = oracle.getrs(LU, ipiv, b)
    xl = scipy.linalg.lu_solve((lu_l, piv_l), b)
    assert np.max(np.abs(x - xl)) / np.max(np.abs(xl)) < 1e-10
    # |L| <= 1
    assert np.max(np.abs(np.tril(LU, -1))) <= 1.0


def test_getrf_backward_error_scale():
    """P A = L U within gamma_n |L||U| componentwise at N=200 (Higham Thm 9.3)."""
    A, _ = oracle.generate(3, 200)
    LU, ipiv, _ = oracle.getrf(A)
    L = np.tril(LU, -1) + np.eye(200)
    Uf = np.triu(LU)
    PA = A[brute.perm_from_ipiv(ipiv, 200)]
    # the product L@U is itself evaluated in floating point: allow gamma_{2n}
    bound = brute.gamma(2 * 200) * (np.abs(L) @ np.abs(Uf))
    assert np.all(np.abs(PA - L @ Uf) <= bound)


def test_rectangular_panel_getrf_vs_lapack():
    """Tall-skinny panel FACT: M x NB panel, LAPACK pivots."""
    rng = np.random.default_rng(9)
    Pn = rng.uniform(-0.5, 0.5, (300, 24))
    LU, ipiv, info = oracle.getrf(Pn)
    p, l, u = scipy.linalg.lu(Pn)  # Pn = p @ l @ u
    lu_l, piv_l = scipy.linalg.lu_factor(Pn)
    assert np.array_equal(ipiv, piv_l.astype(np.int64))
    assert np.allclose(LU, lu_l, rtol=0, atol=1e-13)


# ---------------------------------------------------------------- LASWP / TRSM / GEMM
def test_laswp_vs_permutation():
    """Sequential swaps == gathering by the composed permutation; applying the
    inverse permutation restores A (gather∘scatter identity)."""
    rng = np.random.default_rng(0)
    A = rng.standard_normal((20, 7))
    ipiv = np.array([3, 1, 19, 3, 4, 10, 6], dtype=np.int64)
    S = oracle.laswp(A, 0, 7, ipiv)
    order = brute.perm_from_ipiv(list(ipiv) + list(range(7, 20)), 20)
    assert np.array_equal(S, A[order])
    back = np.empty_like(S)
    back[order] = S
    assert np.array_equal(back, A)
    # column range restriction leaves other columns untouched
    S2 = oracle.laswp(A, 0, 7, ipiv, c0=2, c1=5)
    assert np.array_equal(S2[:, :2], A[:, :2]) and np.array_equal(S2[:, 5:], A[:, 5:])
    assert np.array_equal(S2[:, 2:5], A[order][:, 2:5])


def test_trsm_vs_exact():
    rng = np.random.default_rng(4)
    n, m = 6, 5
    L = np.tril(rng.uniform(-1, 1, (n, n)), -1) + np.eye(n) * 7.0  # diag ignored (unit)
    B = rng.uniform(-1, 1, (n, m))
    X = oracle.trsm_llnu(L, B)
    Lf = brute.to_frac(np.tril(L, -1) + np.eye(n))
    Bf = brute.to_frac(B)
    # exact forward substitution column by column
    for c in range(m):
        y = []
        for i in range(n):
            s = Bf[i][c] - sum(Lf[i][k] * y[k] for k in range(i))
            y.append(s)
        ye = np.array([float(v) for v in y])
        assert np.allclose(X[:, c], ye, rtol=0, atol=1e-13 * max(1, np.abs(ye).max()))
    # closed form: L = I -> X = B exactly
    assert np.array_equal(oracle.trsm_llnu(np.eye(n), B), B)


def test_gemm_update_vs_exact():
    """Each C element within the inner-product bound gamma_k sum|a||b| + u|c| of
    the exact rational value (Higham §3.5)."""
    rng = np.random.default_rng(5)
    m, n, k = 9, 7, 33
    A = rng.uniform(-0.5, 0.5, (m, k))
    B = rng.uniform(-0.5, 0.5, (k, n))
    C = rng.uniform(-0.5, 0.5, (m, n))
    R = oracle.gemm_update(C, A, B)
    Af, Bf, Cf = brute.to_frac(A), brute.to_frac(B), brute.to_frac(C)
    for i in range(m):
        for j in range(n):
            ex = Cf[i][j] - sum(Af[i][p] * Bf[p][j] for p in range(k))
            mag = float(sum(abs(Af[i][p] * Bf[p][j]) for p in range(k)))
            assert abs(R[i, j] - float(ex)) <= brute.gamma(k + 1) * (mag + abs(C[i, j])) + 1e-300
    # zero k-extent / zero A -> C unchanged bitwise
    assert np.array_equal(oracle.gemm_update(C, np.zeros((m, k)), B), C)


def test_maxloc_spec_examples():
    """SPEC.md l.121–123 and l.193–195."""
    assert oracle.maxloc([3.0, 7.0], [5, 2]) == (7.0, 2)
    assert oracle.maxloc([4.0, 4.0], [9, 1]) == (4.0, 1)
    assert oracle.maxloc([1.0, 9.0, 3.0, 9.0], [10, 7, 2, 3]) == (9.0, 3)
    assert oracle.maxloc([2.5], [4]) == (2.5, 4)


# ---------------------------------------------------------------- O3/O4 solves
def test_back_solve_closed_forms():
    """U = I -> x = y; constructed x recovered to 1e-13."""
    y = np.array([1.0, -3.0, 0.5, 2.0])
    x, info = oracle.back_solve(np.eye(4), y)
    assert info == -1 and np.array_equal(x, y)
    rng = np.random.default_rng(8)
    n = 8
    Uu = np.triu(rng.uniform(-0.5, 0.5, (n, n)), 1) + np.diag(rng.uniform(1, 2, n))
    xt = rng.uniform(-1, 1, n)
    # b = U xt computed exactly in rationals then rounded once
    Uf, xf = brute.to_frac(Uu), brute.to_frac(xt)
    b = np.array([float(sum(Uf[i][k] * xf[k] for k in range(n))) for i in range(n)])
    x, info = oracle.back_solve(Uu, b)
    assert np.max(np.abs(x - xt)) < 1e-13
    # zero diagonal -> reported
    Uz = np.eye(3); Uz[1, 1] = 0.0
    assert oracle.back_solve(Uz, np.ones(3))[1] == 1


# ---------------------------------------------------------------- O5 residual
def test_residual_closed_forms():
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    x = np.array([1.0, 2.0])
    b = A @ x  # exact in binary: small integers
    r, parts = oracle.residual(A, x, b)
    assert r == 0.0 and parts[1] == 4.0 and parts[2] == 2.0 and parts[3] == 7.0
    # perturb x by 1e-2 -> >> 16
    assert oracle.residual(A, x + 1e-2, b)[0] > 1e10
    # x = 0 -> resid = ||b|| / (eps * ||b|| * N) = 1 / (eps N)
    r0, _ = oracle.residual(A, np.zeros(2), b)
    assert r0 == pytest.approx(1.0 / (U * 2), rel=1e-15)
    # scale invariance by powers of two (bitwise)
    rng = np.random.default_rng(1)
    A = rng.uniform(-0.5, 0.5, (50, 50)); xx = rng.uniform(-1, 1, 50); bb = rng.uniform(-0.5, 0.5, 50)
    assert oracle.residual(A, xx, bb)[0] == oracle.residual(A * 2.0 ** 7, xx, bb * 2.0 ** 7)[0]


def test_residual_nonfinite_fails():
    """The infinity norm of a vector with a NaN entry is NaN, not the max of
    the other entries: a NaN (or inf) anywhere in x makes the scaled residual
    non-finite, so "resid < 16" fails (a max that skips NaN let
    a NaN solution pass with resid 0)."""
    A = np.array([[2.0, 1.0], [1.0, 3.0]])
    b = A @ np.array([1.0, 2.0])
    for bad in (np.nan, np.inf, -np.inf):
        x = np.array([1.0, bad])
        r, _ = oracle.residual(A, x, b)
        assert not r < 16.0
        x = np.array([bad, 2.0])
        assert not oracle.residual(A, x, b)[0] < 16.0
    A, b = oracle.generate(3, 40)
    x = np.linalg.solve(A, b)
    assert oracle.residual_seeded(40, 3, x)[0] < 16.0
    x[17] = np.nan
    assert not oracle.residual_seeded(40, 3, x)[0] < 16.0


def test_residual_seeded_matches_explicit():
    A, b = oracle.generate(42, 100)
    x = np.linalg.solve(A, b)
    r1, p1 = oracle.residual(A, x, b)
    r2, p2 = oracle.residual_seeded(100, 42, x)
    assert r1 == r2 and np.array_equal(p1, p2)


# ---------------------------------------------------------------- end to end
@pytest.mark.parametrize("N,seed", [(256, 42), (256, 1), (1024, 7)])
def test_oracle_run_passes_hpl(N, seed):
    """HPL invariant: scaled residual < 16 (BASELINE.json); ipiv == LAPACK."""
    r = oracle.run(N, seed)
    assert r["info"] == -1
    assert 0.0 <= r["resid"] < 16.0
    A, b = oracle.generate(seed, N)
    _, piv_l = scipy.linalg.lu_factor(A)
    assert np.array_equal(r["ipiv"], piv_l.astype(np.int64))


def test_oracle_thread_count_invariance():
    """Row-parallel only -> bitwise identical for 1 and many threads."""
    code = ("import oracle,sys,numpy as np; r=oracle.run(300, 5);"
            "sys.stdout.write(r['x'].tobytes().hex()[:4096] + str(r['resid']))")
    outs = []
    for t in ("1", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=t, PYTHONPATH=ROOT)
        outs.append(subprocess.check_output([sys.executable, "-c", code], env=env, cwd=ROOT))
    assert outs[0] == outs[1]


def test_residual_rows_vs_exact():
    """Sampled-row residual (full-size parity helper) vs exact rational sums."""
    N, seed = 40, 9
    A, b = oracle.generate(seed, N)
    x = np.random.default_rng(2).uniform(-1, 1, N)
    rows = np.array([0, 17, 39])
    r, rs = oracle.residual_rows(N, seed, x, rows)
    for t, i in enumerate(rows):
        ex = sum(Fraction(float(A[i, j])) * Fraction(float(x[j])) for j in range(N)) - Fraction(float(b[i]))
        mag = float(sum(abs(Fraction(float(A[i, j])) * Fraction(float(x[j]))) for j in range(N)))
        assert abs(r[t] - float(ex)) <= brute.gamma(N + 1) * (mag + abs(b[i]))
        assert rs[t] == pytest.approx(float(sum(abs(Fraction(float(v))) for v in A[i])), rel=1e-15)
