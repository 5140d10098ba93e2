"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element on the same seeded inputs (-m gpu).  Tolerances are derived in
DESIGN.md §Parity; bit-exact where the step is integer/copy work."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from hpl_inputs import (hpl_panel, integer_panel, random_ipiv, random_unit_lower, twin_panel,
                        upper_well_conditioned)
from tests import brute

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module")
def H():
    import paper_2304_10397_b200 as H
    return H


# ------------------------------------------------------------------ a11 generator
@pytest.mark.parametrize("N,i0,rows,j0,cols", [(256, 0, 256, 0, 257), (8192, 4000, 64, 8100, 93),
                                                (131072, 131000, 72, 131000, 73)])
def test_generator_bitwise(H, N, i0, rows, j0, cols):
    g = H.hplk_generate(42, N, i0, rows, j0, cols)
    o = np.array([[oracle.gen_entry(42, N, i, j) for j in range(j0, j0 + cols)]
                  for i in range(i0, i0 + rows)])
    assert np.array_equal(g, o)


# ------------------------------------------------------------------ a5/a6 DGEMM
def _gemm_tol(A, B, C):
    k = A.shape[1]
    return 2 * brute.gamma(k + 2) * (np.abs(A) @ np.abs(B) + np.abs(C)) + 1e-300


@pytest.mark.parametrize("cfg", [0, 1, 2])
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (128, 64, 16), (300, 200, 64), (513, 257, 37),
                                   (1000, 700, 512), (64, 1, 512), (7, 1031, 256)])
def test_dgemm_update_vs_oracle(H, cfg, m, n, k):
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    A = rng.uniform(-1, 1, (m, k))
    B = rng.uniform(-0.5, 0.5, (k, n))
    C = rng.uniform(-0.5, 0.5, (m, n))
    got = H.hplk_dgemm_update(C, A, B, cfg=cfg)
    ref = oracle.gemm_update(C, A, B)
    assert np.all(np.abs(got - ref) <= _gemm_tol(A, B, C))


def test_dgemm_zero_k_and_identity(H):
    rng = np.random.default_rng(1)
    C = rng.uniform(-1, 1, (50, 40))
    assert np.array_equal(H.hplk_dgemm_update(C, np.zeros((50, 0)), np.zeros((0, 40))), C)
    # A = I (m = k): C - B exactly (one product per element, no rounding beyond the subtract)
    B = rng.uniform(-1, 1, (50, 40))
    assert np.array_equal(H.hplk_dgemm_update(C, np.eye(50), B), C - B)


# ------------------------------------------------------------------ a4 DTRSM
@pytest.mark.parametrize("k,n", [(32, 300), (256, 1000), (512, 129), (13, 5)])
def test_trsm_vs_oracle(H, k, n):
    L = random_unit_lower(k, seed=k)
    rng = np.random.default_rng(n)
    B = rng.uniform(-0.5, 0.5, (k, n))
    got = H.hplk_trsm(L, B)
    ref = oracle.trsm_llnu(L, B)
    # forward error of a triangular solve: <= c k eps cond(L) |X|; L from GEPP,
    # cond_inf(L) measured here, c = 4 (inverse + product)
    Lf = np.tril(L, -1) + np.eye(k)
    cond = np.linalg.norm(Lf, np.inf) * np.linalg.norm(np.linalg.inv(Lf), np.inf)
    tol = 4 * k * U * cond * np.max(np.abs(ref))
    assert np.max(np.abs(got - ref)) <= tol


# ------------------------------------------------------------------ a7 panel FACT
@pytest.mark.parametrize("m,nb,nbmin", [(64, 64, 16), (300, 64, 16), (1000, 256, 16),
                                        (513, 33, 8), (5000, 128, 16), (4096, 512, 16),
                                        (40, 7, 1)])
def test_panel_fact_vs_oracle(H, m, nb, nbmin):
    Pn = hpl_panel(m, nb, seed=m + nb)
    LU, ipiv, info = H.hplk_panel_fact(Pn, nbmin=nbmin)
    LUo, ipo, info_o = oracle.getrf(Pn)
    assert info == -1 and info_o == -1
    assert np.array_equal(ipiv, ipo)
    # factors within 1e-12 elementwise (entries are O(1))
    assert np.max(np.abs(LU - LUo)) <= 1e-12


@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("m,nb,nbmin", [(5000, 128, 16), (777, 64, 16), (3000, 256, 8),
                                        (40, 40, 16), (1200, 96, 4)])
def test_panel_fact_leaf_variants(H, variant, m, nb, nbmin):
    """Left-looking (1) and Crout (2) leaves against the
    oracle, and bitwise against the right-looking leaf (same FMA sequences)."""
    Pn = hpl_panel(m, nb, seed=3 * m + nb)
    LU0, ip0, _ = H.hplk_panel_fact(Pn, nbmin=nbmin)
    LU, ipiv, info = H.hplk_panel_fact(Pn, nbmin=nbmin, leaf_variant=variant)
    LUo, ipo, _ = oracle.getrf(Pn)
    assert info == -1 and np.array_equal(ipiv, ipo)
    assert np.max(np.abs(LU - LUo)) <= 1e-12
    assert np.array_equal(ipiv, ip0) and np.array_equal(LU, LU0)


def test_leaf_variant_end_to_end(H):
    """A whole solve with each leaf variant: pivots and x bitwise equal."""
    def run(v):
        with H.hpl_init(3000, 128, 1, 1, 31) as ctx:
            H.hpl_set_option(ctx, "leaf_variant", v)
            H.hpl_factor(ctx)
            return H.hpl_solve(ctx), H.hpl_get_ipiv(ctx), H.hpl_residual(ctx)
    x0, p0, _ = run(0)
    for v in (1, 2):
        x, p, r = run(v)
        assert np.array_equal(p, p0) and np.array_equal(x, x0) and r < 16


@pytest.mark.parametrize("m,nb,nbmin", [(5000, 128, 16), (777, 64, 16), (26624, 256, 16),
                                        (26625, 64, 16), (300, 33, 8), (40, 40, 16),
                                        (20000, 512, 16)])
def test_panel_fact_cluster_leaf(H, m, nb, nbmin):
    """The one-cluster shared-memory leaf (panels <= 16 x 1664 rows, default)
    against the oracle and bitwise against the grid leaf (leaf_cluster=0)."""
    Pn = hpl_panel(m, nb, seed=7 * m + nb)
    LU1, ip1, info1 = H.hplk_panel_fact(Pn, nbmin=nbmin)
    LU0, ip0, info0 = H.hplk_panel_fact(Pn, nbmin=nbmin, leaf_cluster=0)
    LUo, ipo, _ = oracle.getrf(Pn)
    assert info1 == -1 and info0 == -1 and np.array_equal(ip1, ipo)
    assert np.max(np.abs(LU1 - LUo)) <= 1e-12
    assert np.array_equal(ip1, ip0) and np.array_equal(LU1, LU0)


def test_cluster_leaf_end_to_end(H):
    """A whole solve with the grid leaf only vs the default (cluster leaf for
    small panels): pivots and x bitwise equal."""
    def run(v):
        with H.hpl_init(6000, 256, 1, 1, 37) as ctx:
            H.hpl_set_option(ctx, "leaf_cluster", v)
            H.hpl_factor(ctx)
            return H.hpl_solve(ctx), H.hpl_get_ipiv(ctx), H.hpl_residual(ctx)
    xa, pa, _ = run(0)
    xb, pb, rb = run(1)
    assert np.array_equal(pa, pb) and np.array_equal(xa, xb) and rb < 16


def test_panel_fact_special(H):
    LU, ipiv, info = H.hplk_panel_fact(np.array([[0.0], [3.0]]), nbmin=1)
    assert list(ipiv) == [1] and LU[0, 0] == 3.0 and LU[1, 0] == 0.0 and info == -1
    Pn = hpl_panel(200, 32, seed=5)
    Pn[:, 9] = 0.0     # exact zero column -> singular at 9 (reading A3)
    _, _, info = H.hplk_panel_fact(Pn)
    assert info == 9


LEAVES = [dict(), dict(leaf_cluster=0), dict(leaf_cluster=0, leaf_ctas=3),
          dict(leaf_cluster=0, leaf_ctas=1), dict(leaf_variant=1), dict(leaf_variant=2)]


@pytest.mark.parametrize("leaf", LEAVES, ids=["cluster", "grid", "grid3", "grid1", "left", "crout"])
@pytest.mark.parametrize("m,nb,kind", [(1000, 64, "twin"), (3000, 128, "twin"), (777, 34, "twin"),
                                       (40000, 64, "twin"), (600, 32, "int"), (26000, 64, "int")])
def test_pivot_ties_through_leaves(H, leaf, m, nb, kind):
    """a8 pivot rule (max |v|, ties -> smallest row)
    exercised by the kernels that pick the pivots — the cluster leaf, the
    grid leaf with 1 / 3 / all CTAs, the left-looking and Crout leaves.
    "twin": pairs of rows that are exact negations of each other, far apart
    (different CTAs / cluster ranks), carry every column's maximum; both
    sides update a pair symmetrically, so each pivot is an exact tie and the
    full pivot sequence must equal the oracle's.  "int": small integers, so
    the first column's maximum is shared by many rows across the whole
    panel; only that first pivot is free of rounding (later equalities
    depend on the update's rounding order), so only it is compared."""
    Pn = twin_panel(m, nb, seed=m + nb) if kind == "twin" else integer_panel(m, nb, seed=m)
    LU, ipiv, info = H.hplk_panel_fact(Pn, nbmin=16, **leaf)
    LUo, ipo, info_o = oracle.getrf(Pn)
    if kind == "int":
        first = int(np.flatnonzero(np.abs(Pn[:, 0]) == np.max(np.abs(Pn[:, 0])))[0])
        assert ipiv[0] == ipo[0] == first
        return
    assert info == info_o == -1
    assert np.array_equal(ipiv, ipo), int(np.argmax(ipiv != ipo))
    assert np.max(np.abs(LU - LUo)) <= 1e-12


# ------------------------------------------------------------------ a1/a3 LASWP
@pytest.mark.parametrize("rows,cols,j0,jb,c0,c1", [(300, 200, 0, 32, 32, 200),
                                                   (1000, 513, 256, 256, 1, 513),
                                                   (90, 17, 40, 50, 0, 17),
                                                   (2000, 777, 512, 512, 600, 777)])
def test_laswp_bitwise(H, rows, cols, j0, jb, c0, c1):
    rng = np.random.default_rng(rows + jb)
    A = rng.standard_normal((rows, cols))
    ipiv = random_ipiv(rows, j0, jb, seed=cols)
    A_gpu, Ug = H.hplk_laswp(A, j0, ipiv, c0, c1)
    full_ipiv = np.arange(rows, dtype=np.int64)
    full_ipiv[j0:j0 + jb] = ipiv
    ref = oracle.laswp(A, j0, j0 + jb, full_ipiv, c0, c1)
    assert np.array_equal(Ug, ref[j0:j0 + jb, c0:c1])
    outside = np.ones(rows, bool)
    outside[j0:j0 + jb] = False
    assert np.array_equal(A_gpu[outside][:, c0:c1], ref[outside][:, c0:c1])
    assert np.array_equal(A_gpu[j0:j0 + jb], A[j0:j0 + jb])        # block rows untouched
    assert np.array_equal(A_gpu[:, :c0], A[:, :c0]) and np.array_equal(A_gpu[:, c1:], A[:, c1:])


@pytest.mark.parametrize("rows,cols,NB,P,j0,jb", [(1000, 300, 64, 2, 128, 64), (2000, 517, 32, 4, 64, 32),
                                                  (777, 129, 16, 3, 0, 16), (4096, 1000, 256, 2, 1024, 256),
                                                  (3000, 64, 128, 8, 512, 128)])
def test_rs_exchange_bitwise(H, rows, cols, NB, P, j0, jb):
    """a2/a3: the P > 1 row swaps (rs_gather_peer reading the owners'
    buffers, then rs_scatter) over P emulated process rows give exactly the
    oracle's sequential swaps — bit for bit, pivots that
    cross process rows included."""
    rng = np.random.default_rng(rows + P)
    A = rng.standard_normal((rows, cols))
    ipiv = random_ipiv(rows, j0, jb, seed=cols + P)
    A_gpu, Ug = H.hplk_rs_exchange(A, NB, P, j0, ipiv)
    full_ipiv = np.arange(rows, dtype=np.int64)
    full_ipiv[j0:j0 + jb] = ipiv
    ref = oracle.laswp(A, j0, j0 + jb, full_ipiv)
    assert np.array_equal(Ug, ref[j0:j0 + jb])
    outside = np.ones(rows, bool)
    outside[j0:j0 + jb] = False
    assert np.array_equal(A_gpu[outside], ref[outside])
    assert np.array_equal(A_gpu[j0:j0 + jb], A[j0:j0 + jb])


def test_laswp_identity_moves_nothing(H):
    A = np.random.default_rng(2).standard_normal((64, 40))
    A_gpu, Ug = H.hplk_laswp(A, 8, np.arange(8, 24), 0, 40)
    assert np.array_equal(A_gpu, A) and np.array_equal(Ug, A[8:24])


# ------------------------------------------------------------------ a10 back solve
@pytest.mark.parametrize("N,NB", [(300, 64), (1000, 256), (77, 32), (512, 512), (4000, 128),
                                  (301, 33), (2050, 1024), (3000, 2)])
def test_back_solve_vs_oracle(H, N, NB):
    Uu = upper_well_conditioned(N, seed=N)
    y = np.random.default_rng(N + 1).uniform(-1, 1, N)
    got = H.hplk_back_solve(Uu, y, NB=NB)
    ref, info = oracle.back_solve(Uu, y)
    assert info == -1
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))


# ------------------------------------------------------------------ a11 residual
@pytest.mark.parametrize("N", [256, 3000])
def test_residual_kernel_unit_vectors(H, N):
    """x = e_k: every row of A0 x - b0 is ONE product and one subtraction of
    grid values (exact in binary on both sides), so the device residual rows
    equal the oracle's bit for bit; ||x|| and ||b0|| exact, ||A0|| (a sum of
    N magnitudes, order-dependent) within gamma_N; resid within 2 gamma_N."""
    for k in (0, N // 3, N - 1):
        x = np.zeros(N)
        x[k] = 1.0
        resid, out4, rsum, asum = H.hplk_residual(42, N, x, want_rows=True)
        b = H.hplk_generate(42, N, 0, N, N, 1)[:, 0]
        rows = np.arange(N)
        rr, rowsum = oracle.residual_rows(N, 42, x, rows)
        assert np.array_equal(rsum - b, rr)
        assert np.all(np.abs(asum - rowsum) <= brute.gamma(N) * rowsum)
        ro, po = oracle.residual_seeded(N, 42, x)
        assert out4[0] == po[0] and out4[2] == po[2] == 1.0 and out4[3] == po[3]
        assert abs(out4[1] - po[1]) <= brute.gamma(N) * po[1]
        assert abs(resid - ro) <= 2 * brute.gamma(N) * ro


@pytest.mark.parametrize("N,NB", [(256, 32), (8192, 256)])
def test_residual_vs_oracle_same_x(H, N, NB):
    """SPEC.md l.383-391 two ways on the SAME x: hpl_residual (the ABI call)
    equals the kernel hook bitwise (same kernels), and agrees with the
    oracle's residual of the device x within the bound of two independent
    length-N dot products (|dr_i| <= 2 gamma_{N+1} (sum|a_ij| ||x|| + |b_i|)).
    With x perturbed by 1e-2 the residual has no cancellation:
    both sides agree to 1e-10 relative and fail the < 16 test."""
    with H.hpl_init(N, NB, 1, 1, 42) as ctx:
        H.hpl_factor(ctx)
        x = H.hpl_solve(ctx)
        r_abi = H.hpl_residual(ctx)
    r_k, out4, rsum, asum = H.hplk_residual(42, N, x, want_rows=True)
    assert r_abi == r_k < 16
    ro, po = oracle.residual_seeded(N, 42, x)
    b = H.hplk_generate(42, N, 0, N, N, 1)[:, 0]
    rr, rowsum = oracle.residual_rows(N, 42, x, np.arange(N))
    tol = 2 * brute.gamma(N + 1) * (rowsum * np.max(np.abs(x)) + np.abs(b))
    assert np.all(np.abs((rsum - b) - rr) <= tol)
    assert abs(out4[0] - po[0]) <= np.max(tol)
    assert out4[2] == po[2] and out4[3] == po[3]
    assert abs(out4[1] - po[1]) <= brute.gamma(N) * po[1]
    denom = U * (po[1] * po[2] + po[3]) * N
    assert abs(r_k - ro) <= np.max(tol) / denom + 2 * brute.gamma(N) * ro
    xp = x + 1e-2 * np.random.default_rng(N).uniform(-1, 1, N)
    rp, _ = H.hplk_residual(42, N, xp)
    rpo, _ = oracle.residual_seeded(N, 42, xp)
    assert rp > 1e6 and rpo > 1e6
    assert abs(rp - rpo) <= 1e-10 * rpo


def test_residual_nonfinite_x_fails(H):
    """A NaN or inf anywhere in x makes the device residual +inf (never
    < 16; a max that drops NaN returned 0)."""
    N = 512
    with H.hpl_init(N, 64, 1, 1, 42) as ctx:
        H.hpl_factor(ctx)
        x = H.hpl_solve(ctx)
    for bad in (np.nan, np.inf, -np.inf):
        for k in (0, 300, N - 1):
            xb = x.copy()
            xb[k] = bad
            r, out4 = H.hplk_residual(42, N, xb)
            assert r == np.inf and not r < 16
            assert oracle.residual_seeded(N, 42, xb)[0] >= 16 or \
                np.isnan(oracle.residual_seeded(N, 42, xb)[0])


# ------------------------------------------------------------------ end to end
def _e2e(H, N, NB, seed, lookahead=True):
    with H.hpl_init(N, NB, 1, 1, seed) as ctx:
        H.hpl_set_option(ctx, "lookahead", int(lookahead))
        H.hpl_factor(ctx)
        x = H.hpl_solve(ctx)
        ipiv = H.hpl_get_ipiv(ctx)
        LU = H.hpl_get_local(ctx)
        r = H.hpl_residual(ctx)
    return x, ipiv, LU, r


@pytest.mark.parametrize("N,NB,seed", [(256, 32, 42), (256, 32, 1), (256, 32, 7), (250, 32, 3),
                                       (1000, 64, 42), (2048, 256, 5), (64, 64, 9), (33, 2, 4),
                                       (257, 16, 8)])
def test_hpl_end_to_end_vs_oracle(H, N, NB, seed):
    x, ipiv, LU, r = _e2e(H, N, NB, seed)
    o = oracle.run(N, seed, want_lu=True)
    assert np.array_equal(ipiv, o["ipiv"]), "pivot sequence differs"
    assert np.max(np.abs(x - o["x"])) / np.max(np.abs(o["x"])) <= 1e-9
    assert r < 16.0 and o["resid"] < 16.0
    # U (upper triangle incl. diagonal) is LAPACK-identical up to rounding
    Ug = np.triu(LU[:, :N])
    Uo = np.triu(o["LU"])
    assert np.max(np.abs(Ug - Uo)) <= 1e-10 * max(1.0, np.max(np.abs(Uo)))


def test_lookahead_schedule_invariance(H):
    """the schedule does not change the mathematics."""
    xa, pa, _, _ = _e2e(H, 1024, 64, 11, lookahead=True)
    xb, pb, _, _ = _e2e(H, 1024, 64, 11, lookahead=False)
    assert np.array_equal(pa, pb) and np.array_equal(xa, xb)


def test_split_update_single_gpu_invariance(H):
    """The split update on one GPU: identical pivots and x."""
    def run(split):
        with H.hpl_init(2048, 128, 1, 1, 13) as ctx:
            H.hpl_set_option(ctx, "split", split)
            H.hpl_factor(ctx)
            return H.hpl_solve(ctx), H.hpl_get_ipiv(ctx), H.hpl_residual(ctx)
    xa, pa, ra = run(0)
    xb, pb, rb = run(50)
    assert np.array_equal(pa, pb) and np.array_equal(xa, xb) and rb < 16


@pytest.mark.parametrize("opts", [{"leaf_warp": 148, "leaf_hide_ms": 0},
                                  {"leaf_warp": 7, "leaf_hide_ms": 0},
                                  {"leaf_ctas": 3}, {"leaf_ctas": 0}])
def test_leaf_grid_invariance(H, opts):
    """The leaf's grid (one-warp CTAs beside the DGEMM, few or all multi-warp
    CTAs) only changes which CTA updates a row, never the arithmetic: pivots
    equal the oracle's and x is bitwise that of the default grid."""
    def run(o):
        with H.hpl_init(3000, 128, 1, 1, 17) as ctx:
            for k, v in o.items():
                H.hpl_set_option(ctx, k, v)
            H.hpl_factor(ctx)
            return H.hpl_solve(ctx), H.hpl_get_ipiv(ctx), H.hpl_residual(ctx)
    xa, pa, _ = run({})
    xb, pb, rb = run(opts)
    o = oracle.run(3000, 17)
    assert np.array_equal(pb, o["ipiv"]) and np.array_equal(pa, pb)
    assert np.array_equal(xa, xb) and rb < 16


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_gemm_cfg_end_to_end(H, cfg):
    """Every DGEMM tile config (option gemm_cfg) through hpl_factor: the
    oracle's pivots and x within 1e-9."""
    with H.hpl_init(2048, 128, 1, 1, 43) as ctx:
        H.hpl_set_option(ctx, "gemm_cfg", cfg)
        H.hpl_factor(ctx)
        x, ipiv, r = H.hpl_solve(ctx), H.hpl_get_ipiv(ctx), H.hpl_residual(ctx)
    o = oracle.run(2048, 43)
    assert np.array_equal(ipiv, o["ipiv"]) and r < 16
    assert np.max(np.abs(x - o["x"])) / np.max(np.abs(o["x"])) <= 1e-9


def test_hpl_c1_vs_oracle(H):
    """BASELINE.json configs[1]: N=8192 NB=256 1x1."""
    N, NB, seed = 8192, 256, 42
    x, ipiv, _, r = _e2e(H, N, NB, seed)
    o = oracle.run(N, seed)
    assert np.array_equal(ipiv, o["ipiv"])
    assert np.max(np.abs(x - o["x"])) / np.max(np.abs(o["x"])) <= 1e-9
    assert r < 16.0 and o["resid"] < 16.0


def test_odd_nb_rejected(H):
    """Reading A18: NB must be even (TMA alignment of the L panel)."""
    with pytest.raises(H.HplError) as ei:
        H.hpl_init(100, 33, 1, 1, 1)
    assert ei.value.status == 1


def test_singular_reported(H):
    N = 64
    A = np.random.default_rng(0).uniform(-0.5, 0.5, (N, N + 1))
    A[:, 5] = 0.0
    with H.hpl_init(N, 16, 1, 1, 1) as ctx:
        H.hpl_load_local(ctx, A)
        with pytest.raises(H.HplSingular) as ei:
            H.hpl_factor(ctx)
        assert ei.value.column == 5


def test_load_local_matches_oracle_solve(H):
    """Hand-made system through hpl_load_local (the e2e host path); the
    seeded residual does not apply to it (HPL_ERR_STATE, not a wrong number)."""
    N = 300
    rng = np.random.default_rng(3)
    Ab = rng.uniform(-0.5, 0.5, (N, N + 1))
    with H.hpl_init(N, 32, 1, 1, 1) as ctx:
        H.hpl_load_local(ctx, Ab)
        H.hpl_factor(ctx)
        x = H.hpl_solve(ctx)
        ipiv = H.hpl_get_ipiv(ctx)
        with pytest.raises(H.HplError) as ei:
            H.hpl_residual(ctx)
        assert ei.value.status == 2
        # back to the seeded system: the residual is available again
        H.hpl_regenerate(ctx)
        H.hpl_factor(ctx)
        H.hpl_solve(ctx)
        assert H.hpl_residual(ctx) < 16
    LU, ipo, _ = oracle.getrf(Ab[:, :N])
    xo = oracle.getrs(LU, ipo, Ab[:, N])
    assert np.array_equal(ipiv, ipo)
    assert np.max(np.abs(x - xo)) / np.max(np.abs(xo)) <= 1e-9


@pytest.mark.parametrize("N,NB,pinned", [(3000, 128, True), (8192, 256, True), (1024, 256, False),
                                         (777, 64, True), (8192, 512, True)])
def test_load_factor_bitwise(H, N, NB, pinned):
    """hpl_load_factor (copy overlapped with the first iterations, per-chunk
    streams) gives bitwise the pivots, factors and x of hpl_load_local +
    hpl_factor on the same host system (the seeded one, read back), and
    that system's residual is the seeded residual of the same x."""
    with H.hpl_init(N, NB, 1, 1, 47) as ctx:
        host = H.hpl_get_local(ctx)
        if pinned:
            H.hpl_pin_host(host, True)
        try:
            H.hpl_factor(ctx)
            xa, pa, LUa = H.hpl_solve(ctx), H.hpl_get_ipiv(ctx), H.hpl_get_local(ctx)
            ra = H.hpl_residual(ctx)
            H.hpl_load_factor(ctx, host)
            xb, pb, LUb = H.hpl_solve(ctx), H.hpl_get_ipiv(ctx), H.hpl_get_local(ctx)
            H.hpl_load_factor(ctx, host)          # twice: streams and events reused
            xc = H.hpl_solve(ctx)
        finally:
            if pinned:
                H.hpl_pin_host(host, False)
    assert np.array_equal(pa, pb) and np.array_equal(LUa, LUb)
    assert np.array_equal(xa, xb) and np.array_equal(xa, xc) and ra < 16
    o = oracle.run(N, 47)
    assert np.array_equal(pb, o["ipiv"])


def test_hpl_full_size_c2_sampled(H):
    """BASELINE.json configs[2] (N=131072 NB=512, the bench workload, look-ahead
    on): HPL residual < 16 on the device over all rows, and the oracle's own
    residual on sampled rows (regenerated from the seed, x from the GPU) is
    < 16 too — two independent implementations of the same check."""
    N, NB, seed = 131072, 512, 42
    with H.hpl_init(N, NB, 1, 1, seed) as ctx:
        H.hpl_factor(ctx)
        x = H.hpl_solve(ctx)
        r = H.hpl_residual(ctx)
        ipiv = H.hpl_get_ipiv(ctx)
    assert r < 16.0
    # pivots are valid LAPACK pivots (ipiv[k] >= k) and x is finite
    assert np.all(ipiv >= np.arange(N)) and np.all(ipiv < N)
    assert np.all(np.isfinite(x))
    rows = np.random.default_rng(0).choice(N, 48, replace=False)
    rr, rowsum = oracle.residual_rows(N, seed, x, rows)
    bn = max(abs(oracle.gen_entry(seed, N, i, N)) for i in rows)
    sampled = np.max(np.abs(rr)) / (U * (np.max(rowsum) * np.max(np.abs(x)) + bn) * N)
    assert sampled < 16.0
    # the device residual kernels on the same x: the ABI value bitwise, and
    # the sampled rows elementwise vs the oracle within the dot-product bound
    r_k, out4, rsum, asum = H.hplk_residual(seed, N, x, want_rows=True)
    assert r_k == r
    b = np.array([oracle.gen_entry(seed, N, i, N) for i in rows])
    tol = 2 * brute.gamma(N + 1) * (rowsum * np.max(np.abs(x)) + np.abs(b))
    assert np.all(np.abs((rsum[rows] - b) - rr) <= tol)
    assert np.all(np.abs(asum[rows] - rowsum) <= brute.gamma(N) * rowsum)
