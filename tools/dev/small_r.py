"""Time C1 / C2 PCA runs (one multi-sweep cooperative launch per beta stage) -- dev tool for
the rows-per-thread knob PCA_B200_MULTI_MIN_R."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402

cases = [("c1", P.make_config(64, 64, 2, neighborhood=4, periodic=True, sigma=0.5, beta_period=50, mpm_burn_in=100),
          synth.degrade(synth.smooth_labels(64, 64, 2, 1), 2, 0.5, 2)[None], 200),
         ("c2l5", P.make_config(256, 256, 5, sigma=0.25, mpm_burn_in=750),
          synth.degrade(synth.smooth_labels(256, 256, 5, 3), 5, 0.25, 4)[None], 1000),
         ("c2l9", P.make_config(256, 256, 9, sigma=0.2, mpm_burn_in=750),
          synth.degrade(synth.smooth_labels(256, 256, 9, 3), 9, 0.2, 4)[None], 1000)]
res = {"min_r": os.environ.get("PCA_B200_MULTI_MIN_R", "1")}
for name, cfg, g, n in cases:
    ctx = P.PcaContext(cfg, torch.from_numpy(np.ascontiguousarray(g)).cuda())
    best = 1e30
    for _ in range(3):
        ctx.pca_reset(None, None)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        ctx.pca_sweep(n)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[name] = round(1e3 * best / n, 3)
    ctx.pca_destroy()
print(json.dumps(res))
