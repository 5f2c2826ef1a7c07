"""Time the config-3 sweep for each library variant in build_variants/ (developer tool).
Each variant runs in its own process (PCA_B200_LIB_OVERRIDE)."""
import glob
import json
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
for name, kw in [("moore_torus_mpm", dict(mpm_burn_in=0)), ("moore_torus_nompm", dict(mpm_burn_in=-1)),
                 ("moore_free_mpm", dict(mpm_burn_in=0, periodic=False))]:
    kw2 = dict(neighborhood=8, periodic=True); kw2.update(kw)
    ctx = P.PcaContext(P.make_config(8192, 8192, 2, sigma=0.5, beta0=1.5, beta_step=0, kernel=int(os.environ.get("KSEL", "0")), **kw2), torch.from_numpy(g).cuda())
    ctx.pca_sweep(10); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        ctx.pca_reset(None, None)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream); ctx.pca_sweep(50); b.record(ctx.stream); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 50 * 1e3)
    res[name] = round(best, 2)
    ctx.pca_destroy()
print(json.dumps(res))
'''
out = {}
for lib in sorted(glob.glob(os.path.join(ROOT, "build_variants", os.environ.get("VARIANTS", "packed_*.so")))) + [os.path.join(ROOT, "paper_2507_14869_b200", "libpca_b200.so")]:
    env = dict(os.environ, ROOT=ROOT, PCA_B200_LIB_OVERRIDE=lib)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
    print(os.path.basename(lib), line, flush=True)
