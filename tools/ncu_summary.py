"""Summarise the ncu captures of tools/ncu_kernels.py into a markdown table:
duration, DRAM bytes (read + write), algorithmic bytes / flop of the launch,
achieved rate and fraction of the roofline (HBM: MEASURED_PEAKS.json hbm_gbs;
FP64 tensor: 148 SM x 128 flop/clk x 1965 MHz).

    python tools/ncu_summary.py gpurun_out > profiles/r02_ncu_kernels.md
"""
import csv
import io
import json
import os
import subprocess
import sys

import numpy as np

from hpl_inputs import random_ipiv

d = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
fp64 = 148 * 128 * 1965e6
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
     "launch__registers_per_thread", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"
     ]


def metrics(k):
    out = subprocess.run(["ncu", "-i", os.path.join(d, f"r02_ncu_{k}.ncu-rep"), "--page", "raw",
                          "--csv", "--metrics", ",".join(M)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    r = {}
    for name in M:
        i = h.index(name)
        x = float(v[i].replace(",", ""))
        scale = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1, "us": 1e-6, "ms": 1e-3,
                 "ns": 1e-9, "s": 1.0}.get(u[i], 1.0)
        r[name] = x * scale
    return r


def displaced(rows, j0, jb, ipiv):
    """Rows below the block that receive a block row (index bookkeeping of the
    sequential swaps; the same count the device plan holds)."""
    perm = np.arange(rows)
    for k in range(jb):
        p = ipiv[k]
        perm[[j0 + k, p]] = perm[[p, j0 + k]]
    below = perm[j0 + jb:]
    return int(np.count_nonzero(below != np.arange(j0 + jb, rows)))


n = 32768
ipiv = random_ipiv(n, 4096, 512, seed=1)
nd = displaced(n, 4096, 512, ipiv)
lines = ["# Round 2: ncu captures of the non-DGEMM hot-path kernels", "",
         "One representative launch each (`tools/ncu_kernels.py`, `ncu --set full "
         "--clock-control none -k regex:<kernel> -c 1`, B200, reports in gpurun_out/).",
         f"Rooflines: HBM {hbm / 1e9:.0f} GB/s (MEASURED_PEAKS.json copy bandwidth), "
         f"FP64 tensor {fp64 / 1e12:.2f} TF/s (derived, DESIGN.md §9).", "",
         "| kernel (mode) | launch | time | DRAM R+W | algorithmic | achieved | roofline frac | notes |",
         "|---|---|---|---|---|---|---|---|"]
rows = []
for k, mode, alg, kind, note in [
        ("laswp_gs_kernel", "laswp", 2 * 8 * (512 + nd) * n, "B",
         f"32768 x 32768, jb = 512, {nd} displaced rows: each moved row read + written once"),
        ("rs_gather_peer_kernel", "rs", 2 * 8 * (512 + nd // 2) * n, "B",
         "P = 2 emulated process rows (local memory, not NVLink): U rows + this row's W rows"),
        ("rs_scatter_kernel", "rs", 2 * 8 * (nd // 2) * n, "B", "displaced rows of one process row"),
        ("dgemm_tma_kernel", "trsm", 512 * 512 * 65536, "F",
         "DTRSM as L11^-1 (a_lower ASSIGN) on 512 x 65536; flop = jb^2 n"),
        ("trsm_cols_kernel", "trsm", 512 ** 3 / 3, "F", "L11^-1 by column substitution (per panel)"),
        ("leaf_fact_kernel", "leaf", None, "-", "one 16-column leaf of a 131072 x 512 panel, 8 CTAs"),
        ("bs_partial_kernel", "solve", None, "-", "near sums of one 512-row block (first launch)"),
        ("bs_diag_cluster_kernel", "solve", 8 * 512 * 513 / 2, "B",
         "512 x 512 diagonal block, 16-CTA cluster"),
]:
    try:
        m = metrics(k)
    except Exception as e:  # noqa: BLE001
        lines.append(f"| {k} | - | - | - | - | - | - | no report ({e}) |")
        continue
    t = m["gpu__time_duration.sum"]
    dram = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    if kind == "B":
        ach = alg / t
        cell, frac = f"{ach / 1e9:.0f} GB/s", f"{ach / hbm:.2f} of HBM"
        algs = f"{alg / 1e6:.1f} MB"
    elif kind == "F":
        ach = 2 * alg / t if k == "trsm_cols_kernel" else alg / t
        cell, frac = f"{ach / 1e12:.2f} TF/s", f"{ach / fp64:.2f} of FP64"
        algs = f"{alg / 1e9:.2f} Gflop"
    else:
        cell, frac, algs = "-", "latency-bound", "-"
    extra = (f"DMMA pipe {m['sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active']:.1f} %; "
             if k == "dgemm_tma_kernel" else "")
    lines.append(f"| {k} ({mode}) | {int(m['launch__grid_size'])} CTAs x "
                 f"{int(m['launch__registers_per_thread'])} regs | {t * 1e6:.1f} us | "
                 f"{dram / 1e6:.1f} MB | {algs} | {cell} | {frac} | {extra}warps active "
                 f"{m['sm__warps_active.avg.pct_of_peak_sustained_active']:.0f} %; {note} |")
print("\n".join(lines))
