"""-m gpu: memory-safety checks in place of compute-sanitizer (closed on the GPU pool):

* every kernel family runs on a context whose workspace is followed by a guard band of 0xA5
  bytes, which must be intact afterwards (no write past the caller's workspace);
* run against the debug build (PCA_B200_LIB_OVERRIDE=build_variants/libpca_b200_debug.so,
  built with PCA_DEBUG=1) the same calls also evaluate the kernels' device-side bound checks
  (PCA_DCHECK: ring stage sizes and row ranges of every TMA copy, queue and record indices,
  table-row offsets, decided labels), which trap on violation.

The cases also compare each chain with the oracle, so a run under the debug build is a
parity run of the checked code."""
import os

import numpy as np
import pytest

import oracle as orc
import paper_2507_14869_b200 as P
import synth

pytestmark = pytest.mark.gpu

CASES = [
    # name, H, W, levels, nbhd, periodic, kernel, method, batch
    ("binary TMA ring torus", 40, 1040, 2, 8, True, P.KERNEL_BINARY, "pca", 1),
    ("binary TMA ring free ragged", 37, 1000, 2, 8, False, P.KERNEL_BINARY, "pca", 2),
    ("packed torus", 24, 1024, 2, 8, True, P.KERNEL_PACKED, "pca", 2),
    ("packed free vN", 19, 512, 2, 4, False, P.KERNEL_PACKED, "pca", 1),
    ("table l=5 free", 70, 257, 5, 8, False, P.KERNEL_TABLE, "pca", 2),
    ("table l=3 torus vN", 48, 96, 3, 4, True, P.KERNEL_TABLE, "pca", 1),
    ("general l=9 torus", 40, 130, 9, 8, True, P.KERNEL_GENERAL, "pca", 1),
    ("general l=33 sparse free", 31, 45, 33, 8, False, P.KERNEL_GENERAL, "pca", 1),
    ("Gibbs binary TMA", 32, 1024, 2, 8, True, P.KERNEL_AUTO, "gibbs", 1),
    ("Gibbs quad l=5 free", 30, 77, 5, 8, False, P.KERNEL_AUTO, "gibbs", 1),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0].replace(" ", "_"))
def test_kernels_stay_inside_the_workspace(cuda_device, case):
    name, H, W, L, nb, per, kernel, method, B = case
    g = np.stack([synth.degrade(synth.smooth_labels(H, W, L, 3 + b), L, 0.3, 4 + b) for b in range(B)])
    g[:, ::7, ::5] = synth.random_labels(g[:, ::7, ::5].shape, L, seed=5)  # rare / fp64 sites too
    cfg = P.make_config(H, W, L, batch=B, neighborhood=nb, periodic=per, sigma=0.3, seed=9,
                        mpm_burn_in=1, beta_period=2, kernel=kernel)
    ctx = P.PcaContext(cfg, g, guard=4096)
    m = orc.model(H, W, L, nbhd=nb, periodic=per, sigma=0.3)
    x = g[0].copy()
    for t in range(4):
        (ctx.pca_gibbs_sweep if method == "gibbs" else ctx.pca_sweep)(1)
        beta = orc.beta_at(1.25, 0.25, 2, t)
        x = orc.gibbs_sweep_coloured(m, x, g[0], beta, 9, 0, t) if method == "gibbs" else \
            orc.pca_sweep(m, x, g[0], beta, 9, 0, t)[0]
    assert np.array_equal(ctx.state()[0], x), name
    (ctx.pca_gibbs_sweep if method == "gibbs" else ctx.pca_sweep)(3)  # a run of sweeps per call
    truth = np.stack([synth.smooth_labels(H, W, L, 3 + b) for b in range(B)])
    ctx.pca_finalize(truth, np.zeros_like(truth))
    for kind in (P.EST_LAST, P.EST_MPM, P.EST_MARGINALS, P.EST_CM):
        ctx.estimate(kind)
    if method == "pca":  # (in-place Gibbs sweeps keep no previous state)
        ctx.pca_changed_sites()
        ctx.pca_ssim_windowed(truth, P.EST_MPM)
    ctx.pca_reset(np.ascontiguousarray(g[:, ::-1]), None)
    ctx.pca_sweep(2)
    assert ctx.guard_intact(), f"{name}: a kernel wrote past the workspace"
    ctx.pca_destroy()


def test_debug_build_is_the_library_under_test_when_selected(cuda_device):
    """Under PCA_B200_LIB_OVERRIDE the binding loads that file (the debug build's run)."""
    want = os.environ.get("PCA_B200_LIB_OVERRIDE")
    if want:
        assert os.path.samefile(P.LIB_PATH, want)
