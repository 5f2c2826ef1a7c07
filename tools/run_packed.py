"""ncu target: 8192^2 config-3 sweeps on the packed kernel (developer tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402

burn = int(sys.argv[1]) if len(sys.argv) > 1 else 0
kernel = int(sys.argv[2]) if len(sys.argv) > 2 else P.KERNEL_PACKED
g = torch.from_numpy(synth.degrade(synth.tiled_labels(8192, 8192, 2, 1), 2, 0.5, 2)[None]).cuda()
ctx = P.PcaContext(P.make_config(8192, 8192, 2, periodic=True, sigma=0.5, beta0=1.5, beta_step=0,
                                 mpm_burn_in=burn, kernel=kernel), g)
ctx.pca_sweep(10)
torch.cuda.synchronize()
print("ok")
