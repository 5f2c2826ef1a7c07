"""-m gpu: bench.py's contract line on the real path (short run): every key the driver reads,
consistent values, clocks sampled, launches counted, the roofline filled from a live timing."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_contract_line(cuda_device):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "2", "--warmup", "3", "--sweeps", "8",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
              "gpu_launches", "e2e", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3 and d["value"] > 0
    H, W, S = d["config"]["H"], d["config"]["W"], d["config"]["sweeps_per_step"]
    assert abs(d["value"] - H * W * S / (d["ms_per_step"] * 1e-3)) < 1e-6 * d["value"]
    rf = d["roofline"]
    if d["config"]["kernel"] == "PACKED":  # issue-bound: instructions per SU x SU/s vs the issue peak
        assert rf["bound"] == "alu" and rf["unit"] == "thread-instr/s" and 0 < rf["frac"] < 1.0
        assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
        hb = rf["hbm"]
        assert hb["bound"] == "hbm" and hb["alg_bytes_per_site_update"] == 2.375 and 0 < hb["frac"] < 1.2
    else:
        assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.2
        assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert d["gpu_launches"] >= 2 * (S + 2)
    e2e = d["e2e"]
    # two levels: images cross PCIe bit-packed (packed_io), rows of ceil(W/8) bytes
    assert e2e["h2d_bytes_per_step"] == 2 * H * ((W + 7) // 8)
    assert e2e["d2h_bytes_per_step"] >= H * ((W + 7) // 8) and "packed" in e2e["io"]
    assert 0 < e2e["value"] <= d["value"] * 1.05
    assert d["clocks"]["sm_max_mhz"] > 0
