"""P x Q HPL grid as a single-device loopback (one process, one GPU, one
host thread per rank) through the C ABI — hpl_init_loopback, include/hpl.h.

    python tools/loop_hpl.py N NB P Q [seed] [--oracle] [--la 0|1] [--repeat K]
        [--opt=k=v ...] [--tie] [--absent RANK] [--timeout-ms T] [--load-factor]

Every rank runs the multi-GPU data path (peer-memory RS, pivot exchange,
LBCAST flags, collectives) on the same device, so a 1-GPU box checks rows
a2/a8/a9 (and the split update at P > 1) against the oracle (SURVEY §4
"T-loopback").  --tie loads a hand-made system whose first
panel has exact pivot ties between rows of different process rows
(hpl_inputs.twin_system) and compares with the oracle's GEPP of it.
--absent R: rank R never calls hpl_factor; every other rank must get
HPL_ERR_PEER (bounded waits) instead of hanging.
--load-factor: afterwards every rank runs hpl_load_factor (the pipelined
start: copy overlapped with the first iterations) on its original local
block from pinned host memory; pivots, factors and x must equal the first
run's bitwise.
Prints one JSON line; exit code 0 iff every check passed.
"""
import json
import os
import sys
import time

# Kernels of different ranks wait on each other on one device: they must be
# able to run concurrently (include/hpl.h hpl_init_loopback).  Set before
# the CUDA context exists — this script never imports torch.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    flags = sys.argv[1:]

    def opt(name, default):
        return flags[flags.index(name) + 1] if name in flags else default

    N, NB, P, Q = (int(v) for v in args[:4])
    seed = int(args[4]) if len(args) > 4 and args[4].lstrip("-").isdigit() else 42
    la = int(opt("--la", 1))
    repeat = int(opt("--repeat", 1))
    absent = int(opt("--absent", -1))
    tie = "--tie" in flags
    import paper_2304_10397_b200 as H
    from hpl_inputs import local_block, twin_system

    if os.environ.get("LOOP_WARM"):
        with H.hpl_init(4 * NB, NB, 1, 1, 1) as w:
            H.hpl_factor(w)
            H.hpl_solve(w)
            H.hpl_residual(w)
    ctxs = H.hpl_init_loopback(N, NB, P, Q, seed, 0)
    for c in ctxs:
        H.hpl_set_option(c, "lookahead", la)
        if "--timeout-ms" in flags:
            H.hpl_set_option(c, "peer_timeout_ms", int(opt("--timeout-ms", 20000)))
        for kv in [a for a in flags if a.startswith("--opt=")]:
            k, v = kv[len("--opt="):].split("=")
            H.hpl_set_option(c, k, int(v))
    out = dict(N=N, NB=NB, P=P, Q=Q, seed=seed, mode="loopback", tie=tie)
    ok = True
    try:
        if absent >= 0:
            live = [c for r, c in enumerate(ctxs) if r != absent]
            t0 = time.perf_counter()

            def factor_status(c):
                try:
                    H.hpl_factor(c)
                    return 0, ""
                except H.HplError as e:
                    return e.status, str(e)
            res = H.run_ranks(factor_status, live)
            out["absent"] = absent
            out["statuses"] = [s for s, _ in res]
            out["messages"] = sorted({m for _, m in res})[:2]
            out["wall_s"] = time.perf_counter() - t0
            ok = all(s == 7 for s, _ in res)
            out["peer_error_everywhere"] = ok
            print(json.dumps(out), flush=True)
            return 0 if ok else 1

        Ab = None
        if tie:
            Ab = twin_system(N, NB, P, seed)

        def load(c):
            if Ab is not None:
                r = ctxs.index(c)
                H.hpl_load_local(c, local_block(Ab, NB, P, Q, r % P, r // P))

        for _ in range(repeat - 1):      # earlier factorizations of the same contexts
            H.run_ranks(lambda c: (load(c), H.hpl_factor(c), H.hpl_solve(c, want_x=False),
                                   H.hpl_regenerate(c)), ctxs)
        H.run_ranks(load, ctxs)
        lf = "--load-factor" in flags
        hosts = [H.hpl_get_local(c) for c in ctxs] if lf else None
        t0 = time.perf_counter()
        xs = H.run_ranks(lambda c: (H.hpl_factor(c), H.hpl_solve(c))[1], ctxs)
        out["wall_s"] = time.perf_counter() - t0
        ipivs = [H.hpl_get_ipiv(c) for c in ctxs]
        if lf:
            LUs = [H.hpl_get_local(c) for c in ctxs]
            for h in hosts:
                H.hpl_pin_host(h, True)
            try:
                xb = H.run_ranks(lambda c: (H.hpl_load_factor(c, hosts[ctxs.index(c)]),
                                            H.hpl_solve(c))[1], ctxs)
            finally:
                for h in hosts:
                    H.hpl_pin_host(h, False)
            out["load_factor_bitwise"] = bool(
                all(np.array_equal(a, b) for a, b in zip(xs, xb)) and
                all(np.array_equal(p, H.hpl_get_ipiv(c)) for p, c in zip(ipivs, ctxs)) and
                all(np.array_equal(L, H.hpl_get_local(c)) for L, c in zip(LUs, ctxs)))
            out["pipelined_iters"] = [H.hpl_phase_stats(c).get("pipelined_iters")
                                      for c in ctxs]
            ok = out["load_factor_bitwise"]
            # the loaded system has no seeded residual (HPL_ERR_STATE): back to it
            H.run_ranks(H.hpl_regenerate, ctxs)
            xs = H.run_ranks(lambda c: (H.hpl_factor(c), H.hpl_solve(c))[1], ctxs)
        out["ipiv_replicated"] = all(np.array_equal(ipivs[0], p) for p in ipivs)
        out["x_replicated"] = all(np.array_equal(xs[0], x) for x in xs)
        ok = ok and out["ipiv_replicated"] and out["x_replicated"]
        x, ipiv = xs[0], ipivs[0]
        if not tie:
            rs = H.run_ranks(H.hpl_residual, ctxs)
            out["resid"] = rs[0]
            out["resid_replicated"] = all(r == rs[0] for r in rs)
            ok = ok and rs[0] < 16.0 and out["resid_replicated"]
        out["launches"] = [H.hpl_launch_count(c) for c in ctxs]
        if "--oracle" in flags:
            import oracle
            if tie:
                LU, ipo, info = oracle.getrf(Ab[:, :N])
                xo = oracle.getrs(LU, ipo, Ab[:, N])
                out["oracle_info"] = int(info)
                out["ties_first_panel"] = int(sum(1 for k in range(min(NB, N))
                                                  if ipo[k] != k))
                rr, _ = oracle.residual(Ab[:, :N], x, Ab[:, N])
                out["resid"] = float(rr)
                ok = ok and info == -1 and rr < 16.0
            else:
                o = oracle.run(N, seed)
                ipo, xo = o["ipiv"], o["x"]
                out["oracle_resid"] = o["resid"]
                # the device residual of the device x against the oracle's
                # residual of the same x (two implementations of SPEC.md l.383)
                ro, _ = oracle.residual_seeded(N, seed, x)
                out["oracle_resid_of_gpu_x"] = float(ro)
            out["ipiv_equal"] = bool(np.array_equal(ipiv, ipo))
            if not out["ipiv_equal"]:
                k = int(np.argmax(ipiv != ipo))
                out["first_pivot_mismatch"] = [k, int(ipiv[k]), int(ipo[k])]
            out["x_rel"] = float(np.max(np.abs(x - xo)) / np.max(np.abs(xo)))
            ok = ok and out["ipiv_equal"] and out["x_rel"] <= 1e-9
    except H.HplError as e:
        # who waited for what: every rank's group counters, the arrival flags
        # it received (world and row groups) and its abort detail
        from paper_2304_10397_b200._lib import lib
        dump = {}
        for r, c in enumerate(ctxs):
            buf = np.zeros(4 + 128 + 2, dtype=np.uint64)
            lib.hpl_debug_state(c.h, buf.ctypes.data, len(buf))
            fl = buf[4:132].reshape(4, 32)
            dump[r] = dict(seq=[int(v) for v in buf[:4]],
                           world=[int(v) for v in fl[0, : P * Q]],
                           row=[int(v) for v in fl[1, :Q]], col=[int(v) for v in fl[2, :P]],
                           abort=[int(buf[132]), int(buf[133])])
        out["error"] = str(e)[:400]
        out["debug"] = dump
        ok = False
    finally:
        for c in ctxs:
            H.hpl_free(c)
    out["ok"] = bool(ok)
    print(json.dumps(out), flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
