"""Same-box A/B of library options on one distributed system (one process per
GPU): init once, then for each option set regenerate, factor, solve and
report the device time (max over ranks) and the trailing-DGEMM rate.

    torchrun --nproc-per-node P*Q tools/dist_sweep.py N NB P Q "k=v,k=v" "k=v" ...

An empty string is the default configuration; every set starts from the
defaults.  Runs the list twice (ABAB) to expose box drift."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

DEFAULTS = dict(lookahead=1, leaf_few_ctas=8, leaf_hide_ms=15, split=0,
                leaf_warp=0, leaf_cluster=1, leaf_variant=0)
DIST_DEFAULTS = dict(rs_peer=1, lb_peer=1, fact_gather=65536, fact_gather_ms=8)


def main():
    N, NB, P, Q = (int(v) for v in sys.argv[1:5])
    sets = sys.argv[5:] or [""]
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    import paper_2304_10397_b200 as H
    if world > 1:
        dist.init_process_group("gloo")
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid = torch.frombuffer(bytearray(H.hpl_get_unique_id()), dtype=torch.uint8)
        dist.broadcast(uid, 0)
        ctx = H.hpl_init_dist(N, NB, P, Q, 42, rank, world, bytes(uid.tolist()), local)
    else:
        ctx = H.hpl_init(N, NB, 1, 1, 42)
    H.hpl_set_timing(ctx, True)
    H.hpl_factor(ctx)  # warm-up
    H.hpl_solve(ctx, want_x=False)
    for rep in range(2):
        for sset in sets:
            opts = dict(DEFAULTS, **(DIST_DEFAULTS if world > 1 else {}))
            for kv in filter(None, sset.split(",")):
                k, v = kv.split("=")
                opts[k] = int(v)
            H.hpl_regenerate(ctx)
            for k, v in opts.items():
                H.hpl_set_option(ctx, k, v)
            H.hpl_factor(ctx)
            H.hpl_solve(ctx, want_x=False)
            t = H.hpl_last_timing(ctx)
            r = H.hpl_residual(ctx)
            ms = torch.tensor([t["factor_ms"] + t["solve_ms"]], dtype=torch.float64)
            if world > 1:
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(json.dumps(dict(rep=rep, opts=sset or "default", ms=round(float(ms.item()), 1),
                                      tflops=round((2 / 3 * N ** 3 + 1.5 * N ** 2) / (ms.item() * 1e-3) / 1e12, 3),
                                      dgemm_tf=round(t["dgemm_flop"] / max(t["dgemm_ms"], 1e-9) / 1e9, 2),
                                      resid=r)), flush=True)
    H.hpl_free(ctx)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
