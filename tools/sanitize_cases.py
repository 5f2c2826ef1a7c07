"""Small workloads for compute-sanitizer (memcheck / synccheck / racecheck / initcheck):
every sweep kernel family once, on shapes that run the TMA ring through several stages and
a ragged tail, and the in-place Gibbs kernels.  Each case is also checked against the oracle
so a run under the sanitizer is a parity run too.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as orc  # noqa: E402
import paper_2507_14869_b200 as P  # noqa: E402
import synth  # noqa: E402


def case(name, H, W, L, nb, per, n, gibbs=False, kernel=P.KERNEL_AUTO, batch=1):
    g = np.stack([synth.degrade(synth.smooth_labels(H, W, L, 3 + b), L, 0.3, 4 + b) for b in range(batch)])
    cfg = P.make_config(H, W, L, batch=batch, neighborhood=nb, periodic=per, sigma=0.3, seed=9,
                        mpm_burn_in=1, beta_period=2, kernel=kernel)
    ctx = P.PcaContext(cfg, g)
    m = orc.model(H, W, L, nbhd=nb, periodic=per, sigma=0.3)
    x = g[0].copy()
    for t in range(n):
        (ctx.pca_gibbs_sweep if gibbs else ctx.pca_sweep)(1)
        beta = orc.beta_at(1.25, 0.25, 2, t)
        x = orc.gibbs_sweep_coloured(m, x, g[0], beta, 9, 0, t) if gibbs else \
            orc.pca_sweep(m, x, g[0], beta, 9, 0, t)[0]
    ok = np.array_equal(ctx.state()[0], x)
    truth = np.stack([synth.smooth_labels(H, W, L, 3 + b) for b in range(batch)])
    ctx.pca_finalize(truth, np.zeros_like(truth))
    ctx.pca_destroy()
    print(f"{name}: {'ok' if ok else 'MISMATCH'} (kernel {cfg.kernel})", flush=True)
    return ok


def main():
    good = True
    good &= case("binary TMA ring, torus, 1040 wide", 40, 1040, 2, 8, True, 4)
    good &= case("binary TMA ring, free, ragged 1000 wide", 37, 1000, 2, 8, False, 4)
    good &= case("binary 4-nbr torus 64x64 (multi-sweep path off)", 64, 64, 2, 4, True, 3)
    good &= case("table kernel l=5 free 70x257", 70, 257, 5, 8, False, 4, batch=2)
    good &= case("table kernel l=3 torus 48x96", 48, 96, 3, 4, True, 4)
    good &= case("general kernel l=9 torus 40x130", 40, 130, 9, 8, True, 3)
    good &= case("general kernel l=33 (sparse) free 31x45", 31, 45, 33, 8, False, 3)
    good &= case("Gibbs binary TMA (Moore torus, W%16==0)", 32, 1024, 2, 8, True, 3, gibbs=True)
    good &= case("Gibbs quad kernel l=5 free", 30, 77, 5, 8, False, 3, gibbs=True)
    good &= case("Gibbs fused row parities l=5 torus", 32, 64, 5, 8, True, 3, gibbs=True)
    print("ALL OK" if good else "SOME MISMATCH", flush=True)
    return 0 if good else 1


if __name__ == "__main__":
    os.environ.setdefault("PCA_B200_MULTI_MAX_SITES", "0")  # one launch per sweep: every kernel family
    sys.exit(main())
