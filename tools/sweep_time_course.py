"""Time per sweep along a full paper-protocol run (the cost of the general kernel depends on
how many sites have uniform neighbourhoods, which grows as the chain denoises) -- developer
tool.   python tools/sweep_time_course.py [levels] [batch] [H] [W] [sweeps] [block]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 5
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
H = int(sys.argv[3]) if len(sys.argv) > 3 else 512
W = int(sys.argv[4]) if len(sys.argv) > 4 else 512
n = int(sys.argv[5]) if len(sys.argv) > 5 else 1000
blk = int(sys.argv[6]) if len(sys.argv) > 6 else 100
sig = {2: 0.5, 5: 0.25, 9: 0.2, 33: 0.1}.get(L, 0.25)
g = np.stack([synth.degrade(synth.smooth_labels(H, W, L, 7 + (b % 8)), L, sig, b) for b in range(B)])
cfg = P.make_config(H, W, L, batch=B, sigma=sig, mpm_burn_in=max(0, n - 250))
ctx = P.PcaContext(cfg, torch.from_numpy(g).cuda())
ev = [torch.cuda.Event(enable_timing=True) for _ in range(n // blk + 1)]
ev[0].record(ctx.stream)
for i in range(n // blk):
    ctx.pca_sweep(blk)
    ev[i + 1].record(ctx.stream)
torch.cuda.synchronize()
us = [1e3 * ev[i].elapsed_time(ev[i + 1]) / blk for i in range(n // blk)]
tot = sum(us) * blk
res = {"levels": L, "batch": B, "H": H, "W": W, "sweeps": n, "us_per_sweep_by_block": [round(u, 1) for u in us],
       "mean_us_per_sweep": tot / n, "SU_per_s": B * H * W * n / (tot * 1e-6)}
print(json.dumps(res))
