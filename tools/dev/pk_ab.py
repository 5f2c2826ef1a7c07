"""A/B the packed kernel (dev): us per sweep of 200-sweep calls on 8192^2 (torus Moore MPM on /
off, free Moore on, torus vN on) and the config-4 per-GPU shape 4096 x 32768 (torus, on)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402

out = []
for H, W, nb, per, burn in [(8192, 8192, 8, True, 0), (8192, 8192, 8, True, -1), (8192, 8192, 8, False, 0),
                            (8192, 8192, 4, True, 0), (4096, 32768, 8, True, 0)]:
    g = torch.from_numpy(synth.degrade(synth.tiled_labels(H, W, 2, 1), 2, 0.5, 2)[None]).cuda()
    ctx = P.PcaContext(P.make_config(H, W, 2, neighborhood=nb, periodic=per, sigma=0.5, beta0=1.5, beta_step=0,
                                     mpm_burn_in=burn, kernel=P.KERNEL_PACKED), g)
    ctx.pca_sweep(20)
    best = 1e9
    for _ in range(3):
        ctx.pca_reset(None, None)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream)
        ctx.pca_sweep(200)
        b.record(ctx.stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    out.append(f"{1e3 * best / 200:.1f}")
    ctx.pca_destroy()
print(os.environ.get("PCA_B200_LIB_OVERRIDE", "default").split("/")[-1], " ".join(out), flush=True)
