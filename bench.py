"""bench.py — HPL FP64 TFLOP/s on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                    [--size N] [--block NB] [--no-e2e]

A "step" is one full HPL solve (hpl_factor + hpl_solve: every §8(a) row of
SURVEY.md runs inside it) of the seeded system at the workload size; the
matrix is regenerated on the device between steps (untimed, HPL convention:
generation and the residual check are outside the timing window).  Every
step's scaled residual must be < 16 or the run fails.  Timing: CUDA events on
the library's own streams around factor and solve (hpl_last_timing), summed
over the K steps, max over ranks; inputs (137 GB at the default size) are far
larger than L2.

Default workload at N=1: BASELINE.json configs[2], N=131072 NB=512 on one B200
(the largest single-GPU configuration; configs[1] N=8192 is a parity case).

--impl reference: the CPU oracle (oracle/, plain GEPP) timed on this box's host
cores on a bounded sample of the same workload (a full solve at --cpu-n).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_DERIVED = 148 * 128 * 1965e6 / 1e12  # SMs x FP64 flop/clk x max SM clock (TFLOP/s)


# weak scaling: ~130-137 GB of A per GPU (BASELINE.json configs; 2 GPUs: SURVEY C2b)
N_BY_GPUS = {1: 131072, 2: 185344, 4: 262144, 8: 360448}
GRID_BY_GPUS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}


def workload(a, world: int):
    """(N, NB, P, Q) of this run: --size/--grid, else BASELINE.json's config."""
    n = a.n if a.n > 0 else N_BY_GPUS.get(world, int(131072 * world ** 0.5) // 512 * 512)
    if a.grid:
        P, Q = (int(v) for v in a.grid.lower().split("x"))
    else:
        P, Q = GRID_BY_GPUS.get(world, (1, world))
    assert P * Q == world, f"grid {P}x{Q} needs {P * Q} ranks, have {world}"
    return n, a.nb, P, Q


def cublas_dgemm_tflops(torch) -> float:
    """Library context for the DGEMM roofline: cuBLAS DGEMM 8192^3 through
    torch.matmul(float64), best of 10 (SURVEY.md §8(d) measured-peak (ii))."""
    a = torch.rand(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.rand(8192, 8192, dtype=torch.float64, device="cuda")
    c = torch.matmul(a, b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(10):
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b, c
    torch.cuda.empty_cache()
    return 2 * 8192 ** 3 / (best * 1e-3) / 1e12


def hpl_flops(n: int) -> float:
    return 2.0 / 3.0 * n ** 3 + 1.5 * n ** 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--size", dest="n", type=int, default=0, help="HPL N (0 = weak-scaled default per GPU count)")
    ap.add_argument("--block", dest="nb", type=int, default=512)
    ap.add_argument("--grid", default="", help="PxQ process grid (default: BASELINE.json's grid)")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--cpu-n", type=int, default=8192, help="oracle sample size (C1)")
    ap.add_argument("--ref-n", type=int, default=4096, help="--impl reference: oracle N per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        under = [x for x in sm if x > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(under) if under else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(n: int, seed: int, reps: int = 1):
    """The oracle (plain GEPP + solves) on the host cores: factor+solve of the
    seeded N=n system; returns (TFLOP/s, seconds, threads, resid)."""
    import oracle
    oracle.set_threads(len(os.sched_getaffinity(0)))   # torchrun exports OMP_NUM_THREADS=1
    best = None
    for _ in range(reps):
        A, b = oracle.generate(seed, n)
        t0 = time.perf_counter()
        LU, ipiv, info = oracle.getrf(A)
        x = oracle.getrs(LU, ipiv, b)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    r, _ = oracle.residual_seeded(n, seed, x)
    return hpl_flops(n) / best / 1e12, best, oracle.num_threads(), r


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(a, rank, world):
    """--impl reference: the oracle, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return 0
    for _ in range(a.warmup):
        cpu_baseline(min(a.ref_n, 1024), a.seed)
    times = []
    for _ in range(a.steps):
        tf, dt, thr, r = cpu_baseline(a.ref_n, a.seed)
        if not r < 16.0:
            print(json.dumps({"impl": "reference", "error": f"oracle residual {r}"}))
            return 1
        times.append(dt)
    T = sum(times)
    value = a.steps * hpl_flops(a.ref_n) / T / 1e12
    N, NB, P, Q = workload(a, world)
    line = {
        "impl": "reference",
        "metric": "HPL FP64 TFLOP/s (residual<16)", "value": value, "unit": "TFLOP/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * T / a.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded HPL generator, DESIGN.md reading A6)",
        "config": {"workload": f"HPL N={N} NB={NB} {P}x{Q} grid", "sample": f"full solve at N={a.ref_n}",
                   "N": N, "NB": NB, "grid": f"{P}x{Q}", "l2": "inputs > L2"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": thr, "kind": "oracle",
                         "sample": f"oracle GEPP+solves, full solve at N={a.ref_n} "
                                   f"(bounded sample of the N={N} workload), {cpu_model()}"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return run_reference(a, rank, world)

    import numpy as np
    import torch
    import paper_2304_10397_b200 as H

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")   # rendezvous + scalars; the data path is libhpl (NCCL + peer memory)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def allmax(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    N, NB, P, Q = workload(a, world)
    if world == 1:
        ctx = H.hpl_init(N, NB, 1, 1, a.seed)
    else:
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            uid = torch.frombuffer(bytearray(H.hpl_get_unique_id()), dtype=torch.uint8)
        dist.broadcast(uid, 0)
        # NCCL may print its version on the process's stdout during init: keep
        # stdout for the one JSON line (C-level fd 1 -> fd 2 around the init)
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            ctx = H.hpl_init_dist(N, NB, P, Q, a.seed, rank, world, bytes(uid.tolist()), local)
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    H.hpl_set_timing(ctx, True)
    peak_meas = H.hplk_dmma_peak()
    cublas_tf = cublas_dgemm_tflops(torch)

    fl = hpl_flops(N)
    resids = []
    xs = []

    def step(want_x=False):
        H.hpl_regenerate(ctx)
        barrier()
        H.hpl_factor(ctx)
        x = H.hpl_solve(ctx, want_x=want_x)
        barrier()
        t = H.hpl_last_timing(ctx)
        t["phases"] = H.hpl_phase_stats(ctx)
        r = H.hpl_residual(ctx)
        if not r < 16.0:
            raise SystemExit(f"rank {rank}: HPL residual {r} >= 16 (FAILED)")
        resids.append(r)
        if want_x:
            xs.append(x)
        return t

    for _ in range(a.warmup):
        step()
    clocks = Clocks(local)
    clocks.start()
    # the last timed step also returns x (a 8*N-byte D2H inside its solve):
    # the e2e solve of the same system must reproduce it
    tims = [step(want_x=(k == a.steps - 1)) for k in range(a.steps)]
    ck = clocks.stop()
    dev_ms = sum(t["factor_ms"] + t["solve_ms"] for t in tims)
    dev_ms = allmax(dev_ms)
    dg_ms = sum(t["dgemm_ms"] for t in tims)
    dg_fl = sum(t["dgemm_flop"] for t in tims)
    dg_n = sum(t["dgemm_launches"] for t in tims)
    launches = sum(t["launches"] for t in tims) // max(1, a.steps)
    value = a.steps * fl / (dev_ms * 1e-3) / 1e12   # one P x Q system over all GPUs
    dg_tf = dg_fl / (dg_ms * 1e-3) / 1e12 if dg_ms > 0 else None
    # rooflines of the non-DGEMM phases (summed CUDA-event times over the
    # timed steps, algorithmic bytes / flop from the library: hpl_phase_stats)
    ph = {k: sum(t["phases"][k] for t in tims) for k in tims[0]["phases"]}
    phases = {
        "laswp": {"kernel": "laswp_gs_kernel (P=1) / rs_gather_peer + rs_scatter (P>1), rest columns",
                  "bytes": ph["laswp_bytes"] / a.steps, "ms": ph["laswp_ms"] / a.steps,
                  "GBps": ph["laswp_bytes"] / (ph["laswp_ms"] * 1e-3) / 1e9 if ph["laswp_ms"] > 0 else None,
                  "bound": "hbm"},
        "dtrsm": {"kernel": "dgemm_tma_kernel ASSIGN a_lower (L11^-1 U), rest columns",
                  "flop": ph["trsm_flop"] / a.steps, "ms": ph["trsm_ms"] / a.steps,
                  "TFLOPs": ph["trsm_flop"] / (ph["trsm_ms"] * 1e-3) / 1e12 if ph["trsm_ms"] > 0 else None,
                  "bound": "tensor"},
        "fact": {"kernel": "panel FACT (recursive, device leaf), summed over panels",
                 "ms": ph["fact_ms"] / a.steps, "bound": "latency"},
        "solve": {"kernel": "bs_partial + bs_diag", "bytes": ph["solve_bytes"] / a.steps,
                  "ms": ph["solve_ms"] / a.steps,
                  "GBps": ph["solve_bytes"] / (ph["solve_ms"] * 1e-3) / 1e9 if ph["solve_ms"] > 0 else None,
                  "bound": "hbm"},
    }

    # ---- end to end through the public API with host buffers (pinned)
    e2e = None
    if not a.no_e2e:
        rows, cols = ctx.local_shape
        need = rows * cols * 8
        try:
            avail = int([l for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0].split()[1]) * 1024
        except Exception:
            avail = 0
        local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        if avail < 1.08 * need * local_ranks:
            e2e = {"value": None, "unit": "TFLOP/s", "skipped": f"host RAM {avail / 1e9:.0f} GB < "
                   f"{local_ranks} x {need / 1e9:.0f} GB of local matrices"}
        else:
            host = np.empty((rows, cols), dtype=np.float64)
            H.hpl_regenerate(ctx)
            ctx.check(H.hpl.lib.hpl_get_local(ctx.h, H.hpl.ptr(host), cols))
            pinned = H.hpl_pin_host(host, True)
            xh = np.empty(N, dtype=np.float64)
            barrier()
            t0 = time.perf_counter()
            # the public call that loads and factors: the 137 GB H2D of the
            # local block overlaps the first iterations (hpl_load_factor)
            ctx.check(H.hpl.lib.hpl_load_factor(ctx.h, H.hpl.ptr(host), cols))
            ctx.check(H.hpl.lib.hpl_solve(ctx.h, H.hpl.ptr(xh)))
            barrier()
            dt = allmax(time.perf_counter() - t0)
            # the loaded system is the seeded one (read back after
            # hpl_regenerate): its x must be the verified x of the last
            # timed step (deterministic schedule, bitwise)
            same = bool(np.array_equal(xh, xs[-1]))
            rel = float(np.max(np.abs(xh - xs[-1])) / np.max(np.abs(xs[-1])))
            if not rel <= 1e-12:
                raise SystemExit(f"e2e x differs from the device-path x: {rel}")
            ps = H.hpl_phase_stats(ctx)
            tl = H.hpl_last_timing(ctx)
            e2e = {"value": fl / dt / 1e12, "unit": "TFLOP/s", "x_equal_device_path": same,
                   "api": "hpl_load_factor (H2D overlapped with the first iterations) + hpl_solve",
                   "h2d_ms": ps["h2d_ms"], "h2d_GBps": (ps["h2d_bytes"] / (ps["h2d_ms"] * 1e-3) / 1e9
                                                     if ps["h2d_ms"] > 0 else None),
                   "device_factor_solve_ms": tl["factor_ms"] + tl["solve_ms"],
                   "pipelined_start_ms": ps["pipelined_ms"],
                   "pipelined_iters": ps["pipelined_iters"],
                   "h2d_bytes_per_step": int(rows * cols * 8) * world,
                   "d2h_bytes_per_step": int(N * 8) * world, "pinned": pinned, "s": dt}
            if pinned:
                H.hpl_pin_host(host, False)
            del host

    cpu = None
    if rank == 0 and not a.no_cpu:
        # BASELINE.json configs[0] (C0) and configs[1] (C1): full oracle
        # solves; C1's rate is the reported baseline
        per = {}
        for n_cpu in (256, a.cpu_n):
            tf, dt, thr, rr = cpu_baseline(n_cpu, a.seed)
            per[f"N={n_cpu}"] = {"TFLOPs": tf, "s": dt, "resid": rr}
        cpu = {"value": per[f"N={a.cpu_n}"]["TFLOPs"], "unit": "TFLOP/s", "cores": thr,
               "kind": "oracle",
               "sample": f"oracle GEPP+solves, full solves at N=256 (C0) and N={a.cpu_n} (C1; "
                         f"the value), bounded samples of the N={N} workload, {cpu_model()}",
               "per_config": per}

    traffic, traffic_note = None, None
    tf_path = os.path.join(ROOT, "profiles", "dgemm_traffic.json")
    if os.path.exists(tf_path):
        try:
            tj = json.load(open(tf_path))
            traffic = tj.get("traffic_bytes_per_launch")
            traffic_note = (f"dram read+write per launch at {tj.get('shape')}; algorithmic "
                            f"{tj.get('algorithmic_bytes_per_launch')} B")
        except Exception:
            traffic = None

    H.hpl_free(ctx)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return 0
    line = {
        "metric": "HPL FP64 TFLOP/s (residual<16)",
        "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": dev_ms / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded HPL generator, DESIGN.md reading A6)",
        "config": {"workload": f"HPL N={N} NB={NB} {P}x{Q} grid", "N": N, "NB": NB,
                   "grid": f"{P}x{Q}", "parallelism": "1 GPU" if world == 1 else
                   f"2D block-cyclic {P}x{Q}: LBCAST as copy-engine pulls over NVLink peer memory"
                   " along process rows"
                   + (", pivot search and RS row exchange over NVLink peer memory along process"
                      " columns" if P > 1 else ""),
                   "lookahead": True, "l2": "inputs (~137 GB per GPU) >> L2, no flush needed",
                   "residual_max": max(resids), "frac_of_fp64_peak": value / world / FP64_PEAK_DERIVED},
        "roofline": {"bound": "tensor", "kernel": "dgemm_tma_kernel (trailing update)",
                     "achieved": dg_tf, "peak": FP64_PEAK_DERIVED, "unit": "TFLOP/s",
                     "frac": (dg_tf / FP64_PEAK_DERIVED) if dg_tf else None,
                     "traffic": traffic, "traffic_note": traffic_note,
                     "launches": dg_n // max(1, a.steps),
                     "peak_source": "derived 148 SM x 128 FP64 flop/clk x 1965 MHz (MEASURED_PEAKS"
                                    ".json has no FP64 entry)",
                     "peak_measured_dmma": peak_meas,
                     "cublas_dgemm_8192": cublas_tf},
        "phases": phases,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": ck,
        "impl": "native",
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
