# time the multi-level Gibbs sweep (quad kernel) for each library variant (dev tool)
for lib in build_variants/*.so paper_2507_14869_b200/libpca_b200.so; do
  echo -n "$(basename $lib) "
  PCA_B200_LIB_OVERRIDE=$PWD/$lib python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2507_14869_b200 as P, synth
out = []
for (H, W, L, sig, B) in [(8192, 8192, 5, 0.25, 1), (512, 512, 5, 0.25, 64)]:
    g = np.stack([synth.degrade(synth.tiled_labels(H, W, L, 1), L, sig, 2)] * B)
    ctx = P.PcaContext(P.make_config(H, W, L, batch=B, periodic=True, sigma=sig, beta0=1.5, beta_step=0, mpm_burn_in=0), torch.from_numpy(g).cuda())
    ctx.pca_gibbs_sweep(30); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ctx.stream); ctx.pca_gibbs_sweep(20); b.record(ctx.stream); torch.cuda.synchronize()
    out.append(round(a.elapsed_time(b) / 20 * 1e3, 1))
    ctx.pca_destroy()
print(out)
PY
done
