"""Run one sweep configuration (developer tool, e.g. as an ncu target).
    python tools/run_config.py H W levels sweeps [nbhd periodic mpm kernel method batch]
method: pca (default) or gibbs; batch > 1 tiles the same image over the chains"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402

H, W, L, n = (int(a) for a in sys.argv[1:5])
nb = int(sys.argv[5]) if len(sys.argv) > 5 else 8
per = bool(int(sys.argv[6])) if len(sys.argv) > 6 else True
mpm = int(sys.argv[7]) if len(sys.argv) > 7 else 0
kern = int(sys.argv[8]) if len(sys.argv) > 8 else 0
method = sys.argv[9] if len(sys.argv) > 9 else "pca"
batch = int(sys.argv[10]) if len(sys.argv) > 10 else 1
sig = {2: 0.5, 5: 0.25, 9: 0.2, 33: 0.1}.get(L, 0.25)
import numpy as np  # noqa: E402
g = np.ascontiguousarray(np.repeat(synth.degrade(synth.tiled_labels(H, W, L, 1), L, sig, 2)[None], batch, 0))
ctx = P.PcaContext(P.make_config(H, W, L, batch=batch, neighborhood=nb, periodic=per, sigma=sig,
                                 beta0=1.5, beta_step=0, mpm_burn_in=mpm, kernel=kern),
                   torch.from_numpy(g).cuda())
(ctx.pca_sweep if method == "pca" else ctx.pca_gibbs_sweep)(n)
ctx.pca_sync()
print("ok", ctx.pca_get_stats().sweeps_done)
