"""Multi-GPU parity (-m gpu, needs >= 2 visible GPUs): P x Q grids with one
process per GPU (torchrun), the exchanges over CUDA-IPC peer memory (NCCL
only carries the handle exchange, and the coll_nccl / rs_peer=0 / lb_peer=0
variants), compared with the CPU oracle (identical pivots, x within 1e-9,
residual < 16, x replicated on every rank) — SPEC.md l.363 cross-grid
consistency.  The same data path runs on one GPU in tests/test_loopback.py."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(nproc, N, NB, P, Q, extra=()):
    env = dict(os.environ, PYTHONPATH=ROOT)
    for attempt in range(3):
        # the free port picked here can be taken before torchrun binds it: retry
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
               "--master-port", str(_port()),
               os.path.join(ROOT, "tools", "dist_hpl.py"), str(N), str(NB), str(P), str(Q), "42",
               "--oracle", *extra]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
        if r.returncode == 0 or "EADDRINUSE" not in r.stderr + r.stdout:
            break
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    return json.loads(lines[-1])


@pytest.mark.parametrize("N,NB", [(1024, 64), (2048, 256), (4000, 128)])
def test_1x2_vs_oracle(N, NB):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    out = _run(2, N, NB, 1, 2)
    assert out["ipiv_equal"] and out["x_rel"] <= 1e-9 and out["resid"] < 16


def test_1x2_no_lookahead():
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    out = _run(2, 2048, 128, 1, 2, ("--la", "0"))
    assert out["ipiv_equal"] and out["resid"] < 16


def test_1x4_vs_oracle():
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    out = _run(4, 4096, 256, 1, 4)
    assert out["ipiv_equal"] and out["x_rel"] <= 1e-9 and out["resid"] < 16


@pytest.mark.parametrize("N,NB", [(1024, 64), (2048, 128), (4000, 128)])
def test_2x1_vs_oracle(N, NB):
    """P = 2: distributed pivot search over NVLink peer memory + RS over the
    column communicator."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    out = _run(2, N, NB, 2, 1)
    assert out["ipiv_equal"] and out["x_rel"] <= 1e-9 and out["resid"] < 16


def test_2x1_no_lookahead():
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    out = _run(2, 2048, 128, 2, 1, ("--la", "0"))
    assert out["ipiv_equal"] and out["resid"] < 16


@pytest.mark.parametrize("N,NB,P,Q", [(4096, 256, 2, 2), (3000, 128, 4, 1), (2048, 64, 2, 2)])
def test_4gpu_grids_vs_oracle(N, NB, P, Q):
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    out = _run(4, N, NB, P, Q)
    assert out["ipiv_equal"] and out["x_rel"] <= 1e-9 and out["resid"] < 16


@pytest.mark.parametrize("N,NB,P,Q", [(4096, 256, 2, 4), (4096, 128, 1, 8), (2500, 64, 4, 2)])
def test_8gpu_grids_vs_oracle(N, NB, P, Q):
    if _ngpu() < 8:
        pytest.skip("needs 8 GPUs")
    out = _run(8, N, NB, P, Q)
    assert out["ipiv_equal"] and out["x_rel"] <= 1e-9 and out["resid"] < 16


def test_split_update_schedule_invariance():
    """split update on/off gives the identical pivot sequence
    (P = 2, the RS crossing GPUs; split is off by default)."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    a = _run(2, 3072, 128, 2, 1, ("--opt=split=0",))
    b = _run(2, 3072, 128, 2, 1, ("--opt=split=30",))
    assert a["ipiv_equal"] and b["ipiv_equal"] and a["resid"] < 16 and b["resid"] < 16


@pytest.mark.parametrize("opts", [("--opt=leaf_warp=148", "--opt=leaf_hide_ms=0"),
                                  ("--opt=leaf_warp=5", "--opt=leaf_hide_ms=0")])
def test_2x1_warp_leaf(opts):
    """Distributed leaf as one-warp CTAs (the grid used beside long DGEMMs)."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    out = _run(2, 3000, 128, 2, 1, opts)
    assert out["ipiv_equal"] and out["x_rel"] <= 1e-9 and out["resid"] < 16



@pytest.mark.parametrize("P,Q,split", [(2, 1, 0), (2, 1, 30), (1, 2, 0), (2, 2, 0)])
def test_peer_exchange_vs_nccl(P, Q, split):
    """The RS and LBCAST over NVLink peer memory (defaults: rs_peer=1,
    lb_peer=1) and their NCCL versions (all-reduce + broadcast RS, broadcast
    LBCAST, every collective over NCCL: coll_nccl=1) both give the oracle's
    pivots and x, with and without the split update."""
    if _ngpu() < P * Q:
        pytest.skip(f"needs {P * Q} GPUs")
    for v in (1, 0):
        out = _run(P * Q, 3000, 128, P, Q,
                   (f"--opt=rs_peer={v}", f"--opt=lb_peer={v}", f"--opt=coll_nccl={1 - v}",
                    f"--opt=split={split}"))
        assert out["ipiv_equal"] and out["x_rel"] <= 1e-9 and out["resid"] < 16, (v, out)


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 1), (2, 2)])
def test_load_factor_multi_gpu_bitwise(P, Q):
    """hpl_load_factor across processes (each rank copies its local block in
    column chunks while the first iterations run chunk by chunk; CUDA-IPC
    panel buffers agreed at init): bitwise the LU, pivots and x of
    hpl_load_local + hpl_factor on every rank."""
    if _ngpu() < P * Q:
        pytest.skip(f"needs {P * Q} GPUs")
    out = _run(P * Q, 3000, 64, P, Q, ("--load-factor",))
    assert out["load_factor_bitwise"], out
    assert out["ipiv_equal"] and out["x_rel"] <= 1e-9 and out["resid"] < 16, out


def test_rank_death_gives_peer_error():
    """SPEC.md l.191 / l.360: rank 1 exits 300 ms into hpl_factor; rank 0's
    bounded peer waits end its call with HPL_ERR_PEER instead of a hang.
    (Two plain processes, not torchrun: its agent would kill rank 0 too.)"""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    port = str(_port())
    procs = []
    for rank in (0, 1):
        env = dict(os.environ, PYTHONPATH=ROOT, RANK=str(rank), LOCAL_RANK=str(rank),
                   WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        cmd = [sys.executable, os.path.join(ROOT, "tools", "dist_hpl.py"), "65536", "512", "1",
               "2", "42", "--die", "1:300", "--timeout-ms", "5000"]
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True, env=env))
    outs = [p.communicate(timeout=300) for p in procs]
    lines = [json.loads(l) for l in outs[0][0].splitlines() if l.startswith("{")]
    assert procs[1].returncode == 3, outs[1]
    assert lines and lines[0]["rank"] == 0 and lines[0]["status"] == 7, outs[0]
    assert lines[0]["wall_s"] < 120
