"""Multi-process host logic on CPU (gloo, world_size 2 and 4): the per-rank
iteration plan of the 1 x Q / P x Q block-cyclic driver (hpl_plan_iteration,
the same bookkeeping hpl_factor uses) partitions the trailing columns exactly
and the bench's unique-id exchange round-trips.  No GPU work."""
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


@pytest.mark.parametrize("world,P", [(2, 1), (4, 1), (4, 2)])
def test_plan_partitions_trailing_columns(world, P):
    cases = [(1000, 64), (257, 16), (512, 512), (96, 32)]
    mp.spawn(_worker, args=(world, _free_port(), cases, P), nprocs=world, join=True)
