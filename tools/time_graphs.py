"""Device time per sweep with and without CUDA-graph-captured runs (pca_config.graphs) on
lattices where launch overhead matters (developer tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402

for H, W, B in [(1024, 1024, 1), (2048, 2048, 1), (8192, 8192, 1), (512, 512, 1)]:
    g = torch.from_numpy(synth.degrade(synth.tiled_labels(H, W, 2, 1), 2, 0.5, 2)[None]).cuda()
    for graphs in (0, 1):
        ctx = P.PcaContext(P.make_config(H, W, 2, periodic=True, sigma=0.5, beta0=1.5, beta_step=0,
                                         mpm_burn_in=0, graphs=graphs), g)
        best = 1e9
        for _ in range(4):
            ctx.pca_reset(None, None)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(ctx.stream)
            ctx.pca_sweep(200)
            b.record(ctx.stream)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        st = ctx.pca_get_stats()
        print(f"{H}x{W} kernel {st.kernel} graphs={graphs}: {1e3 * best / 200:.2f} us per sweep "
              f"(replays {st.graph_replays})", flush=True)
        ctx.pca_destroy()
