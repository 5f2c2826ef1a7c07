"""PCA vs Gibbs on the GPU (the run-time comparison PAPER.md:723 calls for) -- developer tool.

    python tools/pca_vs_gibbs.py

For each config: device time per sweep of the synchronous PCA (pca_sweep, one launch per
sweep) and of the checkerboard Gibbs sampler (pca_gibbs_sweep, one launch per colour), and,
Writes gpurun_out/pca_vs_gibbs.json.  The restoration-quality comparison on config 2's
MRF recipe is tests/test_gpu_quality.py (it draws the truths with the oracle's sampler, which
only tests may call).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402


def timed(ctx, method, sweeps):
    run = ctx.pca_sweep if method == "pca" else ctx.pca_gibbs_sweep
    run(min(sweeps, 10))
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        ctx.pca_reset(None, None)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream)
        run(sweeps)
        b.record(ctx.stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def main():
    out = []
    cases = [
        ("c1 64x64 l2 vn4 torus", P.make_config(64, 64, 2, neighborhood=4, periodic=True, sigma=0.5,
                                                 beta_period=50, mpm_burn_in=100),
         synth.degrade(synth.smooth_labels(64, 64, 2, 1), 2, 0.5, 2)[None], 200),
        ("c2 256x256 l5 moore free", P.make_config(256, 256, 5, sigma=0.25, mpm_burn_in=750),
         synth.degrade(synth.smooth_labels(256, 256, 5, 3), 5, 0.25, 4)[None], 1000),
        ("c3 8192x8192 l2 moore torus mpm", P.make_config(8192, 8192, 2, periodic=True, sigma=0.5,
                                                           beta0=1.5, beta_step=0, mpm_burn_in=0),
         synth.degrade(synth.tiled_labels(8192, 8192, 2, 1), 2, 0.5, 2)[None], 50),
        ("c3 8192x8192 l2 moore torus mpm, byte-state PCA kernel (the Gibbs kernel's data path)",
         P.make_config(8192, 8192, 2, periodic=True, sigma=0.5, beta0=1.5, beta_step=0, mpm_burn_in=0,
                       kernel=P.KERNEL_BINARY),
         synth.degrade(synth.tiled_labels(8192, 8192, 2, 1), 2, 0.5, 2)[None], 50),
        ("c3 8192x8192 l5 moore torus mpm", P.make_config(8192, 8192, 5, periodic=True, sigma=0.25,
                                                           beta0=1.5, beta_step=0, mpm_burn_in=0),
         synth.degrade(synth.tiled_labels(8192, 8192, 5, 1), 5, 0.25, 2)[None], 10),
    ]
    for name, cfg, g, sweeps in cases:
        ctx = P.PcaContext(cfg, torch.from_numpy(np.ascontiguousarray(g)).cuda())
        row = {"config": name, "sweeps": sweeps}
        for method in ("pca", "gibbs"):
            ms = timed(ctx, method, sweeps)
            sites = cfg.batch * cfg.height * cfg.width
            row[method] = {"us_per_sweep": 1e3 * ms / sweeps, "SU_per_s": sites * sweeps / (ms * 1e-3)}
        row["gibbs_over_pca_time"] = row["gibbs"]["us_per_sweep"] / row["pca"]["us_per_sweep"]
        print(json.dumps(row), flush=True)
        out.append(row)
        ctx.pca_destroy()

    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open(os.path.join("gpurun_out", "pca_vs_gibbs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
