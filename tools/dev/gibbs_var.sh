# time the two-level Moore Gibbs sweep at 8192^2 for each library variant (dev tool)
for lib in build_variants/*.so paper_2507_14869_b200/libpca_b200.so; do
  echo -n "$(basename $lib) "
  PCA_B200_LIB_OVERRIDE=$PWD/$lib python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2507_14869_b200 as P, synth
g = synth.degrade(synth.tiled_labels(8192, 8192, 2, 1), 2, 0.5, 2)[None]
ctx = P.PcaContext(P.make_config(8192, 8192, 2, periodic=True, sigma=0.5, beta0=1.5, beta_step=0, mpm_burn_in=0), torch.from_numpy(g).cuda())
ctx.pca_gibbs_sweep(5); torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ctx.stream); ctx.pca_gibbs_sweep(30); b.record(ctx.stream); torch.cuda.synchronize()
    best = min(best, a.elapsed_time(b) / 30 * 1e3)
print(round(best, 1))
PY
done
