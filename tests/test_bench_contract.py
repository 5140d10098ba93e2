"""bench.py contract checks that need no GPU: the workload table follows
BASELINE.json's configs (C2 at 1 GPU, C3 2x2 at 4, C4 2x4 at 8; SURVEY §8
C2b at 2), the HPL flop count is the metric's 2/3·N³ + 3/2·N², and the
--impl reference arm (the CPU oracle) prints one well-formed JSON line on
rank 0 and nothing on the other ranks."""
import argparse
import importlib.util
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_workload_matches_baseline_configs():
    b = _bench()
    a = argparse.Namespace(n=0, nb=512, grid="")
    # BASELINE.json configs[2..4] and SURVEY §8 C2b
    assert b.workload(a, 1) == (131072, 512, 1, 1)
    assert b.workload(a, 2) == (185344, 512, 1, 2)
    assert b.workload(a, 4) == (262144, 512, 2, 2)
    assert b.workload(a, 8) == (360448, 512, 2, 4)
    cfg = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert "N=131072 NB=512 1×1" in cfg[2]
    assert "N=262144 NB=512 2×2" in cfg[3]
    assert "N=360448 NB=512 2×4" in cfg[4]
    with pytest.raises(AssertionError):
        b.workload(argparse.Namespace(n=0, nb=512, grid="2x2"), 2)


def test_hpl_flops_formula():
    b = _bench()
    assert b.hpl_flops(1) == pytest.approx(2 / 3 + 1.5)
    n = 131072
    assert b.hpl_flops(n) == pytest.approx(2 * n ** 3 / 3 + 1.5 * n ** 2, rel=1e-15)


def _run_ref(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--steps", "1", "--warmup", "3", "--cpu-n", "512"],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)


def test_reference_arm_json_line():
    p = _run_ref({"RANK": "0", "WORLD_SIZE": "1", "OMP_NUM_THREADS": "2"})
    assert p.returncode == 0, p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("HPL FP64 TFLOP/s") and d["unit"] == "TFLOP/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == 1 and d["warmup"] == 3 and d["dtype"] == "f64"
    assert d["config"]["workload"] == "HPL N=131072 NB=512 1x1 grid"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["value"] == d["value"] and cb["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "TFLOP/s",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_nonzero_rank_is_silent():
    p = _run_ref({"RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0, p.stderr
    assert p.stdout.strip() == ""
