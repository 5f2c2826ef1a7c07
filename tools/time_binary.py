"""Device time per 8192^2 two-level sweep (config 3) for the byte and the bit-packed kernels,
MPM counting on and off (developer tool).
    python tools/time_binary.py [H W]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
g = torch.from_numpy(synth.degrade(synth.tiled_labels(H, W, 2, 1), 2, 0.5, 2)[None]).cuda()
for kernel, name in [(P.KERNEL_BINARY, "byte"), (P.KERNEL_PACKED, "packed")]:
    for burn in (0, -1):
        ctx = P.PcaContext(P.make_config(H, W, 2, periodic=True, sigma=0.5, beta0=1.5, beta_step=0,
                                         mpm_burn_in=burn, kernel=kernel), g)
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
        print(f"{H}x{W} {name:6s} mpm={'on ' if burn == 0 else 'off'}: {1e3 * best / 200:.1f} us per sweep "
              f"(incl. pack/unpack per 200-sweep call)", flush=True)
        ctx.pca_destroy()
