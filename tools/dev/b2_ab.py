"""A/B (dev): us per 8192^2 torus sweep (MPM on) of the byte kernel with one and two sweeps per
pass, and of a Gibbs sweep (checkerboard, binary data path)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402

g = torch.from_numpy(synth.degrade(synth.tiled_labels(8192, 8192, 2, 1), 2, 0.5, 2)[None]).cuda()
out = []
for spp, gibbs in [(1, False), (2, False), (1, True)]:
    ctx = P.PcaContext(P.make_config(8192, 8192, 2, neighborhood=8, periodic=True, sigma=0.5, beta0=1.5, beta_step=0,
                                     mpm_burn_in=0, sweeps_per_pass=spp, kernel=P.KERNEL_BINARY), g)
    run = ctx.pca_gibbs_sweep if gibbs else ctx.pca_sweep
    run(10)
    best = 1e9
    for _ in range(3):
        ctx.pca_reset(None, None)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream)
        run(100)
        b.record(ctx.stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    out.append(f"{1e3 * best / 100:.1f}")
    ctx.pca_destroy()
print(os.environ.get("PCA_B200_LIB_OVERRIDE", "default").split("/")[-1], "byte/pairs/gibbs", " ".join(out), flush=True)
