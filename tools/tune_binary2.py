"""Time config 3 (8192^2 torus, MPM on) with one vs two sweeps per pass for every library
variant in build_variants/ (developer tool)."""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2507_14869_b200 as P, synth
g = synth.degrade(synth.tiled_labels(8192, 8192, 2, 1), 2, 0.5, 2)[None]
res = {}
for spp in (1, 2):
    ctx = P.PcaContext(P.make_config(8192, 8192, 2, neighborhood=8, periodic=True, sigma=0.5, beta0=1.5,
                                     beta_step=0, mpm_burn_in=0, sweeps_per_pass=spp), torch.from_numpy(g).cuda())
    ctx.pca_sweep(10); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        ctx.pca_reset(None, None)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream); ctx.pca_sweep(50); b.record(ctx.stream); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 50 * 1e3)
    res[f"spp{spp}"] = round(best, 2)
    ctx.pca_destroy()
print(json.dumps(res))
'''
for lib in sorted(glob.glob(os.path.join(ROOT, "build_variants", "*.so"))):
    env = dict(os.environ, ROOT=ROOT, PCA_B200_LIB_OVERRIDE=lib)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    print(os.path.basename(lib), line, flush=True)
