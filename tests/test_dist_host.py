"""Multi-process host logic on CPU (gloo, world_size 2, 4 and 8 — the last is
the 2 x 4 grid of BASELINE.json C4): the per-rank iteration plan of the
1 x Q / P x Q block-cyclic driver (hpl_plan_iteration, the same bookkeeping
hpl_factor uses) partitions the trailing columns exactly and the bench's
unique-id exchange round-trips.  No GPU work."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def l2g(l, NB, nprocs, me):
    return ((l // NB) * nprocs + me) * NB + (l % NB)


def _worker(rank, world, port, cases, P):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2304_10397_b200 as H
    Q = world // P
    myrow, mycol = rank % P, rank // P
    for (N, NB) in cases:
        nblk = -(-N // NB)
        for j in range(nblk):
            p = H.hpl_plan_iteration(N, NB, P, Q, myrow, mycol, j)
            mine = [l2g(c, NB, Q, mycol) for r in (p["la"], p["rest"]) for c in range(*r)]
            # only process row 0 contributes (columns are replicated over rows)
            t = torch.zeros(N + 1, dtype=torch.int64)
            if myrow == 0:
                for g in mine:
                    t[g] += 1
            dist.all_reduce(t)
            j0, jb = j * NB, p["jb"]
            want = torch.zeros(N + 1, dtype=torch.int64)
            want[j0 + jb:] = 1
            assert torch.equal(t, want), (N, NB, j)
            # the look-ahead range is panel j+1 on its owner only
            if p["la"][1] > p["la"][0]:
                assert mycol == (j + 1) % Q and p["la"][1] - p["la"][0] == min(NB, N - j0 - jb)
            # the panel's local column exists only on the owner column
            assert (p["lpanel"] >= 0) == (mycol == j % Q)
    # unique-id style byte broadcast (bench.py uses the same gloo path)
    buf = torch.arange(128, dtype=torch.uint8) if rank == 0 else torch.zeros(128, dtype=torch.uint8)
    dist.broadcast(buf, 0)
    assert torch.equal(buf, torch.arange(128, dtype=torch.uint8))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,P", [(2, 1), (4, 1), (4, 2), (8, 2)])
def test_plan_partitions_trailing_columns(world, P):
    cases = [(1000, 64), (257, 16), (512, 512), (96, 32)]
    mp.spawn(_worker, args=(world, _free_port(), cases, P), nprocs=world, join=True)


def _fact_worker(rank, world, port, cases, P, Q):
    """Each rank is one process row of a process column (world == P)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2304_10397_b200 as H
    myrow = rank
    for (N, NB, rows, ms) in cases:
        nblk = -(-N // NB)
        for j in range(nblk):
            f = H.hpl_plan_fact(N, NB, P, Q, myrow, j, rows, ms)
            # the mode is a function of global sizes: every process row agrees
            # (the two FACT paths issue different peer-memory barriers)
            m = torch.tensor([f["mode"]], dtype=torch.int64)
            lo, hi = m.clone(), m.clone()
            dist.all_reduce(lo, op=dist.ReduceOp.MIN)
            dist.all_reduce(hi, op=dist.ReduceOp.MAX)
            assert lo.item() == hi.item() == f["mode"], (N, NB, j)
            # closed form of the switch
            M = N - j * NB
            rest_ms = 2.0 * -(-M // P) * -(-M // Q) * NB / 35e12 * 1e3
            want = 1 if (rows > 0 and M <= min(rows, min(N, 1 << 16)) and rest_ms <= ms) else 0
            assert f["mode"] == want and f["rows"] == M, (N, NB, j, f)
            # the combined panel [T; every row's L rows] covers each global row
            # of the panel exactly once: the gather kernel's row map is onto
            jb = min(NB, M)
            t = torch.zeros(N, dtype=torch.int64)
            for i in range(f["mL"]):
                g = l2g(f["lrL0"] + i, NB, P, myrow)
                t[g] += 1
            if myrow == j % P:      # T (block row j) is counted once, on its owner
                t[j * NB:j * NB + jb] += 1
            dist.all_reduce(t)
            want_t = torch.zeros(N, dtype=torch.int64)
            want_t[j * NB:] = 1
            assert torch.equal(t, want_t), (N, NB, j)
            # lrL0 + mL = the local row count, ldp covers jb + mL rows, 16-aligned
            mloc = sum(min(NB, N - b * NB) for b in range(myrow, nblk, P))
            assert f["lrL0"] + f["mL"] == mloc
            assert f["ldp"] >= jb + f["mL"] and f["ldp"] % 16 == 0
    dist.destroy_process_group()


@pytest.mark.parametrize("P,Q", [(2, 1), (2, 2), (2, 4), (4, 1)])
def test_fact_plan_agrees_across_the_column(P, Q):
    cases = [(1000, 64, 65536, 8.0), (3000, 128, 1500, 1e9), (4099, 256, 65536, 1e-6),
             (131072, 4096, 65536, 8.0)]
    mp.spawn(_fact_worker, args=(P, _free_port(), cases, P, Q), nprocs=P, join=True)


def test_fact_plan_single_process_mode():
    import paper_2304_10397_b200 as H
    assert H.hpl_plan_fact(1000, 64, 1, 1, 0, 3)["mode"] == -1
    with pytest.raises(H.HplError):
        H.hpl_plan_fact(1000, 64, 2, 1, 2, 0)
