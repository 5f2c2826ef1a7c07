"""Fraction of sites whose Moore neighbourhood is uniform / two-label / other along a
paper-protocol run (what decides the general kernel's integer vs fp64 paths) -- dev tool."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402


def mix(x):
    H, W = x.shape
    nb = [x[1 + dr:H - 1 + dr, 1 + dc:W - 1 + dc] for dr in (-1, 0, 1) for dc in (-1, 0, 1)
          if (dr, dc) != (0, 0)]
    nb = np.stack(nb)
    uni = (nb == nb[0]).all(0)
    s2 = np.where(nb != nb[0], nb, 255).min(0)
    two = ((nb == nb[0]) | (nb == s2)).all(0) & ~uni
    return float(uni.mean()), float(two.mean()), float(1 - uni.mean() - two.mean())


for L, sig in [(5, 0.25), (9, 0.2), (33, 0.1)]:
    truth = synth.smooth_labels(512, 512, L, 7)
    g = synth.degrade(truth, L, sig, 1)
    ctx = P.PcaContext(P.make_config(512, 512, L, sigma=sig), torch.from_numpy(g[None].copy()).cuda())
    out = {"levels": L}
    for upto in (0, 100, 600, 1000):
        ctx.pca_sweep(upto - ctx.pca_get_stats().sweeps_done)
        out[f"sweep{upto}"] = [round(v, 3) for v in mix(ctx.state()[0])]
    out["truth"] = [round(v, 3) for v in mix(truth)]
    print(json.dumps(out), flush=True)
