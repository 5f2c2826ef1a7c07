"""CPU checks of bench.py's contract that need no GPU: the reference arm (the oracle, timed on
the host) prints one JSON line with the keys the driver reads, and the workload recipe."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(300)
def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_workloads():
    sys.path.insert(0, ROOT)
    import bench
    w1 = bench.workload(1)
    assert (w1["H"], w1["W"], w1["rows"], w1["levels"]) == (8192, 8192, 8192, 2)
    w8 = bench.workload(8)
    assert (w8["H"], w8["W"], w8["rows"]) == (32768, 32768, 4096)  # config 4 at P = 8
    assert bench.BYTES_PER_SU == 7 and bench.BYTES_PER_SU_PACKED == 2.375


@pytest.mark.timeout(300)
def test_multi_gpu_self_launch_reaches_the_strip_path_dry_run():
    """`python bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (the driver's
    scaling run); --dry-run does the ranks' orchestration on CPU (gloo, stub context): the
    config-4 workload for N = 2, each rank's 4096-row strip, the ring neighbours, the NCCL
    unique id broadcast, and one line from rank 0."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=280,
                       env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["dry_run"] is True and d["n_gpus"] == 2
    assert d["config"]["H"] == 8192 and d["config"]["W"] == 32768
    ranks = sorted(d["ranks"], key=lambda e: e["rank"])
    assert [(e["row0"], e["rows"]) for e in ranks] == [(0, 4096), (4096, 4096)]
    assert [(e["up"], e["down"]) for e in ranks] == [(1, 1), (0, 0)]  # a 2-rank ring (torus)
    assert all(e["unique_id_bytes"] == 128 for e in ranks)


def test_strong_scaling_dry_run_splits_the_32768_lattice():
    """`--scaling strong` (SURVEY 8(d) C4's secondary mode): the 32768^2 torus split over the
    ranks, 16384 rows each at N = 2, and the line says strong."""
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run", "--scaling", "strong",
                        "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=280, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip().startswith("{")][0])
    assert d["scaling"] == "strong" and d["config"]["H"] == 32768 and d["config"]["W"] == 32768
    assert sorted((e["row0"], e["rows"]) for e in d["ranks"]) == [(0, 16384), (16384, 16384)]
