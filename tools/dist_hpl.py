"""Multi-rank HPL through the C ABI (one process per GPU).

    torchrun --nproc-per-node Q --master-addr 127.0.0.1 --master-port PORT \\
        tools/dist_hpl.py N NB P Q [seed] [--oracle] [--la 0|1] [--repeat K] [--opt=k=v]
        [--die RANK:MS] [--timeout-ms T] [--load-factor]

rank 0 creates the NCCL unique id (hpl_get_unique_id); it travels to the other
ranks over a gloo process group; every rank then calls hpl_init_dist.  With
--oracle, rank 0 compares the pivots and x with the CPU oracle.
--load-factor: every rank then runs hpl_load_factor (pipelined start) on its
original local block; LU, pivots and x must equal the first run's bitwise.
Prints one JSON line on rank 0; exit code 0 iff residual < 16 (and parity).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    N, NB, P, Q = (int(v) for v in args[:4])
    seed = int(args[4]) if len(args) > 4 else 42
    la = 1
    if "--la" in sys.argv:
        la = int(sys.argv[sys.argv.index("--la") + 1])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_2304_10397_b200 as H
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid = torch.frombuffer(bytearray(H.hpl_get_unique_id()), dtype=torch.uint8)
    dist.broadcast(uid, 0)
    ctx = H.hpl_init_dist(N, NB, P, Q, seed, rank, world, bytes(uid.tolist()), local)
    H.hpl_set_option(ctx, "lookahead", la)
    for kv in [a for a in sys.argv[1:] if a.startswith("--opt=")]:
        k, v = kv[len("--opt="):].split("=")
        H.hpl_set_option(ctx, k, int(v))
    if "--timeout-ms" in sys.argv:
        H.hpl_set_option(ctx, "peer_timeout_ms", int(sys.argv[sys.argv.index("--timeout-ms") + 1]))
    if "--die" in sys.argv:
        # failure detection: rank R exits MS ms into
        # hpl_factor; every other rank must get HPL_ERR_PEER, not hang
        die_rank, die_ms = (int(v) for v in sys.argv[sys.argv.index("--die") + 1].split(":"))
        if rank == die_rank:
            import threading
            threading.Timer(die_ms / 1000.0, lambda: os._exit(3)).start()
        dist.barrier()
        t0 = time.perf_counter()
        try:
            H.hpl_factor(ctx)
            H.hpl_solve(ctx)
            status, msg = 0, ""
        except H.HplError as e:
            status, msg = e.status, str(e)
        print(json.dumps(dict(rank=rank, status=status, msg=msg[:300],
                              wall_s=time.perf_counter() - t0)), flush=True)
        os._exit(0 if status == 7 else 1)
    timeline = "--timeline" in sys.argv
    repeat = int(sys.argv[sys.argv.index("--repeat") + 1]) if "--repeat" in sys.argv else 1
    for _ in range(repeat - 1):      # earlier factorizations of the same context
        H.hpl_factor(ctx)
        H.hpl_solve(ctx, want_x=False)
        H.hpl_regenerate(ctx)
    if timeline:
        H.hpl_set_timing(ctx, True)
        H.hpl_factor(ctx)            # warm-up pass
        H.hpl_regenerate(ctx)
    dist.barrier()
    t0 = time.perf_counter()
    H.hpl_factor(ctx)
    x = H.hpl_solve(ctx)
    dist.barrier()
    wall = time.perf_counter() - t0
    tm = H.hpl_last_timing(ctx)
    if timeline:
        tl = H.hpl_get_timeline(ctx)
        fd = H.hpl_get_fact_detail(ctx)
        fact, la_, rest, lsw, trsm, dg = tl.T
        summ = dict(rank=rank, factor_ms=round(tm["factor_ms"], 1), sum_fact=round(fact.sum(), 1),
                    sum_la=round(la_.sum(), 1), sum_rest=round(rest.sum(), 1),
                    sum_rs=round(lsw.sum(), 1), sum_trsm=round(trsm.sum(), 1),
                    sum_dgemm=round(dg.sum(), 1),
                    dgemm_tflops=round(tm["dgemm_flop"] / max(tm["dgemm_ms"], 1e-9) / 1e9, 2),
                    fact_iter0=round(float(fact[0]), 2), rest_iter0=round(float(rest[0]), 2),
                    sum_fact_wait=round(float(fd[:, 0].sum()), 1),
                    sum_fact_local=round(float(fd[:, 1].sum()), 1),
                    sum_lbcast_plan=round(float(fd[:, 2].sum()), 1),
                    fact_local_iter0=round(float(fd[0, 1]), 2),
                    lbcast_plan_iter0=round(float(fd[0, 2]), 2))
        print(json.dumps(summ), flush=True)
        for a in sys.argv[1:]:
            if a.startswith("--timeline-out="):
                np.savetxt(f"{a.split('=', 1)[1]}_r{rank}.csv", np.hstack([tl, fd]), delimiter=",",
                           fmt="%.4f", header="fact,la_update,rest_update,rest_rs,rest_trsm,"
                           "rest_dgemm,fact_wait,fact_local,lbcast_plan")
    ipiv = H.hpl_get_ipiv(ctx)
    lf_ok = True
    if "--load-factor" in sys.argv:
        # the pipelined start (copy overlapped with the first iterations) on
        # this rank's original local block: bitwise the same LU, pivots and x
        LU = H.hpl_get_local(ctx)
        H.hpl_regenerate(ctx)
        host = H.hpl_get_local(ctx)
        H.hpl_pin_host(host, True)
        H.hpl_load_factor(ctx, host)
        xb = H.hpl_solve(ctx)
        H.hpl_pin_host(host, False)
        lf_ok = bool(np.array_equal(x, xb) and np.array_equal(ipiv, H.hpl_get_ipiv(ctx)) and
                     np.array_equal(LU, H.hpl_get_local(ctx)) and
                     H.hpl_phase_stats(ctx)["pipelined_iters"] > 0)
        H.hpl_regenerate(ctx)         # the seeded system again, for the residual
        H.hpl_factor(ctx)
        H.hpl_solve(ctx, want_x=False)
    r = H.hpl_residual(ctx)
    H.hpl_free(ctx)
    dev = torch.tensor([tm["factor_ms"] + tm["solve_ms"]], dtype=torch.float64)
    dist.all_reduce(dev, op=dist.ReduceOp.MAX)
    ok = r < 16.0
    out = dict(N=N, NB=NB, P=P, Q=Q, resid=r, wall_s=wall, device_ms=float(dev.item()),
               tflops=(2 / 3 * N ** 3 + 1.5 * N ** 2) / (float(dev.item()) * 1e-3) / 1e12)
    if "--oracle" in sys.argv and rank == 0:
        import oracle
        o = oracle.run(N, seed)
        out["ipiv_equal"] = bool(np.array_equal(ipiv, o["ipiv"]))
        out["x_rel"] = float(np.max(np.abs(x - o["x"])) / np.max(np.abs(o["x"])))
        out["oracle_resid"] = o["resid"]
        ok = ok and out["ipiv_equal"] and out["x_rel"] <= 1e-9 and o["resid"] < 16.0
    # every rank must hold the same x and pivots
    xs = torch.from_numpy(x.copy())
    x0 = xs.clone()
    dist.broadcast(x0, 0)
    out_same = bool(torch.equal(xs, x0))
    flag = torch.tensor([1 if out_same else 0], dtype=torch.int64)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    out["x_replicated"] = bool(flag.item())
    ok = ok and out["x_replicated"]
    if "--load-factor" in sys.argv:
        f2 = torch.tensor([1 if lf_ok else 0], dtype=torch.int64)
        dist.all_reduce(f2, op=dist.ReduceOp.MIN)
        out["load_factor_bitwise"] = bool(f2.item())
        ok = ok and out["load_factor_bitwise"]
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
