"""Multi-GPU data path on ONE GPU (-m gpu): P x Q grids as a single-device
loopback (hpl_init_loopback: P*Q rank contexts in one process, one host
thread each; tools/loop_hpl.py), compared with the CPU oracle.

Every rank runs the same kernels, flags and schedule as on P*Q GPUs — the
peer-memory RS row gather (§8 a2), the pivot search across the
process column (a8), the LBCAST flag/pull protocol (a9,
PAPER.md l.6/l.9), the split update (f1) and the
collectives — only the peer pointers are the sibling contexts' instead of
CUDA-IPC mappings.  Checks: identical pivot sequence to the oracle, x within
1e-9 (BASELINE.json), x / pivots / residual replicated on every rank,
residual < 16 (SPEC.md l.187-213, l.363 cross-grid consistency).  Each case
runs in its own process (the loopback needs CUDA_MODULE_LOADING=EAGER and
32 hardware queues before CUDA initialises) under a timeout.

The P*Q ranks share one GPU, and their kernels wait on each other: nothing
guarantees the device co-schedules them (B200_PROFILING.md), and in stress
runs ~1-3 % of 8-rank runs hit a bounded peer wait (HPL_ERR_PEER) —
DESIGN.md §6.2 lists what was measured and removed.  A case that ends with
HPL_ERR_PEER is therefore run once more; a wrong pivot, a wrong x, a CUDA
error or a second timeout fails."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(N, NB, P, Q, *extra, seed=42, expect_ok=True):
    env = dict(os.environ, PYTHONPATH=ROOT, CUDA_MODULE_LOADING="EAGER",
               CUDA_DEVICE_MAX_CONNECTIONS="32")
    cmd = [sys.executable, os.path.join(ROOT, "tools", "loop_hpl.py"), str(N), str(NB), str(P),
           str(Q), str(seed), "--oracle", *extra]
    for attempt in range(2):
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        assert lines, r.stdout[-3000:] + r.stderr[-3000:]
        out = json.loads(lines[-1])
        # one more run only for a co-scheduling timeout of the shared GPU
        if not (expect_ok and "HPL_ERR_PEER" in out.get("error", "")
                and "HPL_ERR_CUDA" not in out.get("error", "")):
            break
        out["retried_after_peer_timeout"] = True
    if expect_ok:
        assert r.returncode == 0 and out.get("ok", out.get("peer_error_everywhere")), \
            out.get("error", out)
    return out


def _check(out):
    assert out["ipiv_equal"], out
    assert out["x_rel"] <= 1e-9, out
    assert out["x_replicated"] and out["ipiv_replicated"], out


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 1), (2, 2), (4, 1), (2, 4)])
@pytest.mark.parametrize("N,NB", [(1024, 64), (3000, 128)])
def test_loopback_grid_vs_oracle(N, NB, P, Q):
    """Grids 1x2, 2x1, 2x2, 4x1 and 2x4 (BASELINE.json C4's grid shape)."""
    out = _run(N, NB, P, Q)
    _check(out)
    assert out["resid"] < 16 and out["resid_replicated"]


@pytest.mark.parametrize("P,Q", [(2, 1), (2, 2)])
def test_loopback_split_update(P, Q):
    """The split update with the RS crossing process rows:
    RS_L(j) overlaps UPDATE_R(j); identical pivots and x within 1e-9."""
    _check(_run(3000, 128, P, Q, "--opt=split=30"))


@pytest.mark.parametrize("rs_peer,lb_peer", [(1, 1), (0, 1), (1, 0), (0, 0)])
def test_loopback_exchange_variants(rs_peer, lb_peer):
    """RS as the peer-memory row gather or as the collective variant (U
    all-reduced, W broadcast); LBCAST as copy-engine pulls or a broadcast."""
    _check(_run(3000, 128, 2, 2, f"--opt=rs_peer={rs_peer}", f"--opt=lb_peer={lb_peer}"))


@pytest.mark.parametrize("P,Q", [(2, 1), (2, 2)])
@pytest.mark.parametrize("gather", [0, 1 << 20, 1500])
def test_loopback_fact_modes(P, Q, gather):
    """P > 1 panel FACT: the distributed leaf (fact_gather=0: one pivot
    exchange per column over peer memory), the gathered FACT (every panel),
    and a threshold that switches mode mid-run."""
    _check(_run(3000, 128, P, Q, f"--opt=fact_gather={gather}", "--opt=fact_gather_ms=100000"))


def test_loopback_distributed_leaf_one_warp_ctas():
    """The distributed leaf as one-warp CTAs (the grid used beside long DGEMMs)."""
    _check(_run(3000, 128, 2, 1, "--opt=fact_gather=0", "--opt=leaf_warp=8",
                "--opt=leaf_hide_ms=0"))


def test_loopback_no_lookahead():
    _check(_run(2048, 128, 2, 2, "--la", "0"))


def test_loopback_two_factorizations():
    """Flags and collective counters are monotonic across factorizations of
    one context (hpl_regenerate, then a second hpl_factor)."""
    _check(_run(2048, 64, 2, 2, "--repeat", "2"))


@pytest.mark.parametrize("P,Q", [(1, 1), (2, 1), (2, 2), (4, 1)])
def test_loopback_cross_row_pivot_ties(P, Q):
    """SPEC.md l.118 / l.194: exact ties between rows of DIFFERENT process
    rows (hpl_inputs.twin_system) are won by the smaller global row, as in
    the oracle's GEPP of the same hand-made system."""
    out = _run(1024, 64, P, Q, "--tie", "--opt=fact_gather=0")
    _check(out)
    assert out["ties_first_panel"] > 0 and out["resid"] < 16
    # and through the gathered FACT
    _check(_run(1024, 64, P, Q, "--tie", "--opt=fact_gather=1048576",
                "--opt=fact_gather_ms=100000"))


def test_loopback_absent_rank_times_out():
    """SPEC.md l.191 / l.360: a rank that never enters hpl_factor makes every
    other rank's call return HPL_ERR_PEER (bounded device waits), not hang."""
    out = _run(1024, 64, 2, 2, "--absent", "3", "--timeout-ms", "2000")
    assert out["peer_error_everywhere"] and out["statuses"] == [7, 7, 7], out
    assert out["wall_s"] < 60


@pytest.mark.parametrize("P,Q,extra", [(1, 2, ()), (2, 1, ()), (2, 2, ()), (2, 4, ()),
                                       (2, 2, ("--opt=split=30",)),
                                       (2, 2, ("--opt=rs_peer=0", "--opt=lb_peer=0")),
                                       (2, 2, ("--opt=fact_gather=1048576",
                                               "--opt=fact_gather_ms=100000"))])
def test_loopback_load_factor_bitwise(P, Q, extra):
    """hpl_load_factor on a grid (the pipelined start: every rank copies its
    local block in column chunks while the first K iterations run chunk by
    chunk, FACT/LBCAST of panels 0..K in chunk 0, per-chunk RS barriers
    within the process column): pivots, factors and x bitwise those of
    hpl_load_local + hpl_factor on every rank; then the seeded system again
    vs the oracle."""
    out = _run(3000, 64, P, Q, "--load-factor", *extra)
    _check(out)
    assert out["load_factor_bitwise"], out
    assert all(k == 6 for k in out["pipelined_iters"]), out


@pytest.mark.parametrize("N,NB,P,Q", [(100, 64, 2, 4), (64, 64, 2, 2), (130, 64, 4, 1), (2, 2, 1, 2),
                                      (33, 32, 2, 2), (66, 32, 2, 4), (200, 64, 1, 4),
                                      (129, 64, 2, 1), (513, 64, 4, 2), (4, 2, 2, 2)])
def test_loopback_degenerate_grids(N, NB, P, Q):
    """Grids where some ranks own no matrix rows or no columns (N=100 on 2x4:
    process columns 2 and 3 hold nothing; N=NB: one block; ragged last
    blocks of 1-2 rows/columns; N=2 and 4): every rank still takes part in
    every collective and the result is the oracle's."""
    _check(_run(N, NB, P, Q))
