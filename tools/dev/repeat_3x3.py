"""Repeat the 3x3 torus lockstep case many times, after a large-lattice context, to look
for nondeterminism (developer tool)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402
from parity_helpers import lockstep, make_ctx  # noqa: E402

bad = 0
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 50):
    if it % 10 == 0:  # dirty the caching allocator with a big context
        big = make_ctx(P.make_config(64, 64, 2, neighborhood=4, periodic=True, sigma=0.3, seed=it),
                       synth.random_labels((64, 64), 2, it))
        big.pca_sweep(3)
        del big
    H, W, L, nb, per = 3, 3, 2, 8, True
    cfg = P.make_config(H, W, L, neighborhood=nb, periodic=per, sigma=0.3, beta0=0.9,
                        beta_step=0.5, beta_period=2, seed=1234 + H * W)
    g = synth.random_labels((H, W), L, seed=H * 1000 + W)
    x0 = synth.random_labels((H, W), L, seed=W * 1000 + H)
    ctx = make_ctx(cfg, g, x0)
    t = lockstep(ctx, cfg, 6)
    if t.mismatches:
        bad += 1
        print("iteration", it, "mismatches", t.mismatches, "margin", t.max_margin, flush=True)
print("bad", bad)
