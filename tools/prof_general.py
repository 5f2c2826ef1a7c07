"""Run a multi-level workload to a chosen sweep and open the profiler around ONE sweep launch
(developer tool, the ncu target for the general kernel's captures):

    ncu --profile-from-start off --set full --import-source on -c 1 -o out \
        python tools/prof_general.py c5 900
    python tools/prof_general.py c5 900 --time      # no profiler: us per sweep around t

workloads: c5     128 chains x 512^2, l = 5, Moore-8, free boundary, paper schedule, MPM
                  burn-in 750 (SURVEY 8(d) C5 per GPU)
           l5big  8192^2, l = 5, Moore-8 torus, fixed beta 1.5, MPM every sweep (C3 l = 5)
           c2     256^2, l = 5, Moore-8 free, paper schedule, burn-in 750 (one launch per sweep
                  is forced with rows_per_thread so the capture is a plain sweep launch)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402


KERNEL = 0


def workload(name):
    if name == "c5":
        B = 128
        g = np.stack([synth.degrade(synth.smooth_labels(512, 512, 5, 7), 5, 0.25, s) for s in range(B)])
        return P.make_config(512, 512, 5, batch=B, sigma=0.25, mpm_burn_in=750, kernel=KERNEL), g
    if name == "l5big":
        g = synth.degrade(synth.tiled_labels(8192, 8192, 5, 1), 5, 0.25, 2)[None]
        return P.make_config(8192, 8192, 5, periodic=True, sigma=0.25, beta0=1.5, beta_step=0,
                             mpm_burn_in=0, kernel=KERNEL), g
    if name == "c2_33":  # config 2's 33-level image (256^2, Moore free, sigma 0.1); small: the
        # runtime runs each beta stage's sweeps in one cooperative launch (sweep_multi_kernel)
        g = synth.degrade(synth.smooth_labels(256, 256, 33, 3), 33, 0.1, 4)[None]
        return P.make_config(256, 256, 33, sigma=0.1, mpm_burn_in=750, kernel=KERNEL), g
    raise SystemExit(f"unknown workload {name}")


def main():
    global KERNEL
    name, t = sys.argv[1], int(sys.argv[2])
    if "--kernel" in sys.argv:
        KERNEL = int(sys.argv[sys.argv.index("--kernel") + 1])
    cfg, g = workload(name)
    ctx = P.PcaContext(cfg, torch.from_numpy(np.ascontiguousarray(g)).cuda())
    # one launch per sweep (the runtime splits pca_sweep(n) into per-sweep launches here)
    ctx.pca_sweep(t)
    torch.cuda.synchronize()
    if "--time" in sys.argv:
        n = 20
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream)
        ctx.pca_sweep(n)
        b.record(ctx.stream)
        torch.cuda.synchronize()
        print(f"{name} t={t} kernel={ctx.pca_get_stats().kernel}: {1e3 * a.elapsed_time(b) / n:.1f} us "
              f"per sweep", flush=True)
        return
    torch.cuda.profiler.start()
    ctx.pca_sweep(1)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("ok", ctx.pca_get_stats().sweeps_done, flush=True)


if __name__ == "__main__":
    main()
