import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_sessionstart(session):
    """Build the in-tree CUDA library when it is missing or older than its sources (a no-op
    otherwise), so the ABI and GPU tests always load the current code."""
    from paper_2507_14869_b200 import build as B

    B.build()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("-m gpu test run without a CUDA device")
    return torch.device("cuda:0")


def pytest_sessionfinish(session, exitstatus):
    """Parity report: per test, the site updates compared with the oracle in lockstep, the
    near-tie mismatches and the largest oracle margin of a mismatch (north star / R19)."""
    import json

    helpers = sys.modules.get("parity_helpers") or sys.modules.get("tests.parity_helpers")
    if helpers is None or not helpers.REGISTRY:
        return
    rep = {}
    for t in helpers.REGISTRY:
        e = rep.setdefault(t.name, {"updates": 0, "mismatches": 0, "max_margin": 0.0})
        e["updates"] += t.updates
        e["mismatches"] += t.mismatches
        e["max_margin"] = max(e["max_margin"], t.max_margin)
    tot_u = sum(e["updates"] for e in rep.values())
    tot_m = sum(e["mismatches"] for e in rep.values())
    out = {"tolerance": {"margin": 1e-6, "rate": 1e-6},
           "total": {"updates": tot_u, "mismatches": tot_m,
                     "rate": tot_m / tot_u if tot_u else 0.0,
                     "max_margin": max(e["max_margin"] for e in rep.values())},
           "tests": rep}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "parity_report.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
