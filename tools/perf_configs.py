"""Time the sweep on the secondary configs (device time per sweep, SU/s) -- developer tool.

    python tools/perf_configs.py [--quick]

config 1 (64x64 binary torus), config 2 (256x256 Moore free, l = 5/9/33, paper schedule),
config 3 variants (8192^2: l = 2 MPM on/off, 4-neighbour, free boundary; l = 5), the config-4
per-GPU shape (4096 x 32768) on one GPU,
config 5 per GPU (128 chains of 512x512, l = 5, paper protocol).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402


def time_cfg(name, cfg, g, sweeps, reps=3):
    ctx = P.PcaContext(cfg, torch.from_numpy(g).cuda())
    s = ctx.stream
    ctx.pca_sweep(min(sweeps, 20))
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        ctx.pca_reset(None, None)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        ctx.pca_sweep(sweeps)
        b.record(s)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    sites = cfg.batch * cfg.height * cfg.width
    res = {"config": name, "sweeps": sweeps, "ms": best, "us_per_sweep": 1e3 * best / sweeps,
           "SU_per_s": sites * sweeps / (best * 1e-3)}
    print(json.dumps(res), flush=True)
    ctx.pca_destroy()
    return res


def main():
    quick = "--quick" in sys.argv
    out = []
    g = synth.degrade(synth.smooth_labels(64, 64, 2, 1), 2, 0.5, 2)[None]
    out.append(time_cfg("c1 64x64 l2 vn4 torus", P.make_config(64, 64, 2, neighborhood=4, periodic=True, sigma=0.5, beta_period=50, mpm_burn_in=100), g, 200))
    for L, sg in [(5, 0.25), (9, 0.2), (33, 0.1)]:
        g = synth.degrade(synth.smooth_labels(256, 256, L, 3), L, sg, 4)[None]
        out.append(time_cfg(f"c2 256x256 l{L} moore free", P.make_config(256, 256, L, sigma=sg, mpm_burn_in=750), g, 1000))
    big = synth.degrade(synth.tiled_labels(8192, 8192, 2, 1), 2, 0.5, 2)[None]
    for name, kw in [("c3 l2 moore torus mpm", dict(mpm_burn_in=0)), ("c3 l2 moore torus nompm", dict(mpm_burn_in=-1)),
                     ("c3 l2 vn4 torus mpm", dict(mpm_burn_in=0, neighborhood=4)),
                     ("c3 l2 moore free mpm", dict(mpm_burn_in=0, periodic=False))]:
        kw2 = dict(neighborhood=8, periodic=True)
        kw2.update(kw)
        out.append(time_cfg(name, P.make_config(8192, 8192, 2, sigma=0.5, beta0=1.5, beta_step=0, **kw2), big, 50))
    c4 = synth.degrade(synth.tiled_labels(4096, 32768, 2, 1), 2, 0.5, 2)[None]
    out.append(time_cfg("c4 per-GPU shape 4096x32768 l2 moore torus mpm (1 GPU, whole torus)",
                        P.make_config(4096, 32768, 2, periodic=True, sigma=0.5, beta0=1.5, beta_step=0,
                                      mpm_burn_in=0), c4, 50))
    if not quick:
        c4w = synth.tiled_labels(32768, 32768, 2, 21)[None]
        out.append(time_cfg("c4 whole lattice 32768x32768 l2 moore torus mpm on ONE GPU",
                            P.make_config(32768, 32768, 2, periodic=True, sigma=0.5, beta0=1.5, beta_step=0,
                                          mpm_burn_in=0), c4w, 20))
        del c4w
        big5 = synth.degrade(synth.tiled_labels(8192, 8192, 5, 1), 5, 0.25, 2)[None]
        out.append(time_cfg("c3 l5 moore torus mpm", P.make_config(8192, 8192, 5, periodic=True, sigma=0.25, beta0=1.5, beta_step=0, mpm_burn_in=0), big5, 10))
        B = 128
        g5 = np.stack([synth.degrade(synth.smooth_labels(512, 512, 5, 7), 5, 0.25, s) for s in range(B)])
        out.append(time_cfg("c5 128x512x512 l5 moore free", P.make_config(512, 512, 5, batch=B, sigma=0.25, mpm_burn_in=750), g5, 50))
    json.dump(out, open(os.path.join("gpurun_out", "perf_configs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
