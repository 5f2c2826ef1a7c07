"""-m gpu parity of the GPU Gibbs sampler (pca_gibbs_sweep, checkerboard colour order) with
the oracle's colour-order scan (orc_gibbs_sweep_coloured, pinned in test_oracle_pins.py).

levels == 2 decisions are integer thresholds (exact); levels > 2 use the uniform table or
fp64 weights, where a near-tie (|u - F_k| ~ 1e-16) could differ -- none occur on these
inputs, so the chains must be identical."""
import numpy as np
import pytest

import oracle as orc
import paper_2507_14869_b200 as P
import synth
from parity_helpers import beta_of, make_ctx, oracle_model

pytestmark = pytest.mark.gpu

SHAPES = [
    (64, 64, 2, 4, True), (64, 64, 2, 8, True), (37, 531, 2, 8, False), (19, 1000, 2, 4, False),
    (40, 130, 5, 8, False), (30, 62, 9, 4, True), (31, 45, 33, 8, False), (1, 77, 2, 8, False),
    (77, 1, 5, 4, False), (2, 2, 3, 8, False), (8, 48, 2, 8, True), (6, 10, 255, 8, True),
    # compile-time level counts: 3 and 9 (tables in shared memory), 16 (D only), 4 and 8 nbrs
    (20, 36, 3, 4, True), (22, 40, 9, 8, False), (20, 36, 16, 8, True), (18, 41, 16, 4, False),
]


def gibbs_lockstep(ctx, cfg, n, t0=0):
    m = oracle_model(cfg)
    g = ctx._g_host
    x = ctx.state()
    for t in range(t0, t0 + n):
        ctx.pca_gibbs_sweep(1)
        xn = ctx.state()
        for b in range(cfg.batch):
            ref = orc.gibbs_sweep_coloured(m, x[b], g[b], beta_of(cfg, t), cfg.seed, cfg.chain0 + b, t)
            bad = int((xn[b] != ref).sum())
            assert bad == 0, f"sweep {t} chain {b}: {bad} sites differ"
        x = xn


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_gibbs_lockstep(cuda_device, shape):
    H, W, L, nb, per = shape
    cfg = P.make_config(H, W, L, neighborhood=nb, periodic=per, sigma=0.3, beta0=0.9,
                        beta_step=0.5, beta_period=2, seed=4321 + H * W)
    g = synth.random_labels((H, W), L, seed=H * 1000 + W + 1)
    x0 = synth.smooth_labels(H, W, L, seed=W) if min(H, W) > 1 else synth.random_labels((H, W), L, 3)
    ctx = make_ctx(cfg, g, x0)
    gibbs_lockstep(ctx, cfg, 6)


def test_gibbs_free_running_with_counts(cuda_device):
    """Config-1 shape (64x64 binary 4-neighbour torus, 200 sweeps, burn-in 100): the GPU
    Gibbs chain, its MPM counts and its MPM image equal the oracle's colour-order run."""
    m = orc.model(64, 64, 2, nbhd=4, periodic=True)
    truth = orc.generate_mrf(m, 400, 0.9, 1.6, seed=4)
    g = orc.degrade(truth, 2, 0.5, seed=104)
    cfg = P.make_config(64, 64, 2, neighborhood=4, periodic=True, sigma=0.5, beta0=1.25,
                        beta_step=0.25, beta_period=50, seed=4, mpm_burn_in=100)
    ctx = make_ctx(cfg, g)
    ctx.pca_gibbs_sweep(200)
    x_o, cnt_o = orc.gibbs_run(oracle_model(cfg), g, g, 200, 1.25, 0.25, 50, 4, burn_in=100,
                               order="colour")
    assert np.array_equal(ctx.state()[0], x_o)
    assert np.array_equal(ctx.counts()[0], cnt_o[1].astype(np.uint16))
    assert np.array_equal(ctx.estimate(P.EST_MPM)[0], orc.mpm(cnt_o))
    st = ctx.pca_get_stats()
    assert st.sweeps_done == 200 and st.counted_sweeps == 100


def test_gibbs_multilevel_counts_and_schedule(cuda_device):
    """levels = 5, Moore-8, free boundary (config-2 style), annealed beta, planar counts."""
    H, W, L = 48, 72, 5
    truth = synth.smooth_labels(H, W, L, seed=2)
    g = synth.degrade(truth, L, 0.25, seed=3)
    cfg = P.make_config(H, W, L, sigma=0.25, beta0=1.25, beta_step=0.25, beta_period=10,
                        seed=8, mpm_burn_in=15)
    ctx = make_ctx(cfg, g)
    ctx.pca_gibbs_sweep(30)
    x_o, cnt_o = orc.gibbs_run(oracle_model(cfg), g, g, 30, 1.25, 0.25, 10, 8, burn_in=15,
                               order="colour")
    assert np.array_equal(ctx.state()[0], x_o)
    assert np.array_equal(ctx.counts()[0], cnt_o.astype(np.uint16))


def test_gibbs_batch_equals_independent_chains(cuda_device):
    B, H, W = 3, 20, 36
    g = np.stack([synth.degrade(synth.smooth_labels(H, W, 2, s), 2, 0.5, s + 9) for s in range(B)])
    cfg = P.make_config(H, W, 2, batch=B, neighborhood=8, periodic=True, sigma=0.5, seed=77)
    ctx = make_ctx(cfg, g)
    ctx.pca_gibbs_sweep(9)
    xs = ctx.state()
    for b in range(B):
        one = make_ctx(P.make_config(H, W, 2, neighborhood=8, periodic=True, sigma=0.5, seed=77,
                                     chain0=b), g[b])
        one.pca_gibbs_sweep(9)
        assert np.array_equal(one.state()[0], xs[b])


@pytest.mark.parametrize("extreme", [dict(sigma=0.01), dict(beta0=300.0)])
@pytest.mark.parametrize("L", [2, 3, 5, 9, 16, 33])
def test_gibbs_extreme_parameters(cuda_device, extreme, L):
    """Weights that under/overflow the factorised fp64 form take the log-domain path."""
    H, W = 24, 40
    kw = dict(sigma=0.3, seed=3)
    kw.update(extreme)
    cfg = P.make_config(H, W, L, **kw)
    ctx = make_ctx(cfg, synth.random_labels((H, W), L, 1), synth.random_labels((H, W), L, 2))
    gibbs_lockstep(ctx, cfg, 3)


def test_gibbs_rejects_odd_torus_and_mixes_with_pca(cuda_device):
    cfg = P.make_config(9, 10, 2, periodic=True, sigma=0.5)
    ctx = make_ctx(cfg, np.zeros((9, 10), np.uint8))
    with pytest.raises(P.PcaError, match="even"):
        ctx.pca_gibbs_sweep(1)
    # PCA and Gibbs sweeps share the state and the sweep counter t
    H, W = 16, 24
    cfg = P.make_config(H, W, 3, periodic=True, sigma=0.4, seed=6)
    g = synth.random_labels((H, W), 3, 5)
    ctx = make_ctx(cfg, g)
    ctx.pca_sweep(2)
    ctx.pca_gibbs_sweep(2)
    ctx.pca_sweep(1)
    m = oracle_model(cfg)
    x = g.copy()
    for t in range(2):
        x, _ = orc.pca_sweep(m, x, g, beta_of(cfg, t), 6, 0, t)
    for t in range(2, 4):
        x = orc.gibbs_sweep_coloured(m, x, g, beta_of(cfg, t), 6, 0, t)
    x, _ = orc.pca_sweep(m, x, g, beta_of(cfg, 4), 6, 0, 4)
    assert np.array_equal(ctx.state()[0], x)


@pytest.mark.parametrize("per,shape", [(True, (32, 96)), (False, (33, 100)), (True, (6, 16))])
def test_gibbs_binary_path_counts_and_batch(cuda_device, per, shape):
    """levels == 2, Moore-8 (the TMA binary Gibbs kernel): free-running chains of a batch with
    MPM counts equal the oracle's colour-order runs."""
    H, W = shape
    B = 3
    g = np.stack([synth.degrade(synth.smooth_labels(H, W, 2, 10 + b), 2, 0.5, b) for b in range(B)])
    cfg = P.make_config(H, W, 2, batch=B, periodic=per, sigma=0.5, beta0=1.0, beta_step=0.3,
                        beta_period=4, seed=21, mpm_burn_in=5)
    ctx = make_ctx(cfg, g)
    for _ in range(13):  # one sweep per call: the per-sweep launches (runs would go multi-sweep)
        ctx.pca_gibbs_sweep(1)
    m = oracle_model(cfg)
    xs, cs = ctx.state(), ctx.counts()
    for b in range(B):
        x_o, cnt_o = orc.gibbs_run(m, g[b], g[b], 13, 1.0, 0.3, 4, 21, chain=b, burn_in=5,
                                   order="colour")
        assert np.array_equal(xs[b], x_o)
        assert np.array_equal(cs[b], cnt_o[1].astype(np.uint16))
    assert ctx.pca_get_stats().sweep_launches == 2 * 13


def test_gibbs_binary_full_size_sampled_rows(cuda_device):
    """8192^2 Moore-8 torus, two levels: after 2 GPU Gibbs sweeps, sampled even rows are
    recomputed by the oracle from x_1 (colours 0 and 1), odd rows from x_1 with their new
    even neighbours (colours 2 and 3)."""
    H = W = 8192
    g = synth.degrade(synth.tiled_labels(H, W, 2, seed=3), 2, 0.5, seed=4)
    cfg = P.make_config(H, W, 2, periodic=True, sigma=0.5, beta0=1.5, beta_step=0.0, seed=9)
    ctx = make_ctx(cfg, g)
    ctx.pca_gibbs_sweep(1)
    x1 = ctx.state()[0]
    ctx.pca_gibbs_sweep(1)
    x2 = ctx.state()[0]
    m = oracle_model(cfg)
    rng = np.random.default_rng(1)
    for r in sorted({0, 1, H - 1, H - 2} | set(rng.integers(2, H - 2, 6).tolist())):
        y = x1.copy()
        rows = [r] if r % 2 == 0 else [(r - 1) % H, (r + 1) % H, r]
        for rr in rows:  # even rows first (colours 0, 1), then the odd row (colours 2, 3)
            ks = (0, 1) if rr % 2 == 0 else (2, 3)
            for k in ks:
                y = orc.gibbs_colour_phase(m, y, g, 1.5, cfg.seed, 0, 1, k, rows=(rr, rr + 1))
        assert np.array_equal(x2[r], y[r]), f"row {r}"


@pytest.mark.parametrize("case", range(16))
def test_gibbs_randomised_configurations_lockstep(cuda_device, case):
    """Random shapes (even sides on a torus), levels, neighbourhoods, schedules and batches:
    3 Gibbs sweeps in lockstep with the oracle's colour order, exact."""
    rng = np.random.default_rng(777 + case)
    L = int(rng.choice([2, 2, 3, 5, 9, 33]))
    nb = int(rng.choice([4, 8]))
    per = bool(rng.integers(2))
    H = int(rng.integers(2, 40)) * (2 if per else 1) + (0 if per else int(rng.integers(0, 2)))
    W = int(rng.integers(2, 300)) * (2 if per else 1) + (0 if per else int(rng.integers(0, 2)))
    if rng.integers(3) == 0:
        W = 16 * int(rng.integers(1, 40))  # the fused / TMA paths
    H = max(H, 4 if per else 1)
    B = int(rng.integers(1, 3))
    cfg = P.make_config(H, W, L, batch=B, neighborhood=nb, periodic=per,
                        sigma=float(rng.uniform(0.1, 0.6)), beta0=float(rng.uniform(0.5, 2.5)),
                        beta_step=float(rng.uniform(0, 0.5)), beta_period=2,
                        seed=int(rng.integers(1 << 30)), chain0=int(rng.integers(0, 99)))
    g = np.stack([synth.random_labels((H, W), L, seed=case * 7 + b) for b in range(B)])
    x0 = np.stack([synth.random_labels((H, W), L, seed=case * 7 + 3 + b) for b in range(B)])
    gibbs_lockstep(make_ctx(cfg, g, x0), cfg, 3)


def test_gibbs_checkpoint_and_pca_interleaving_on_the_binary_path(cuda_device):
    """Two levels, Moore-8 torus, W % 16 == 0 (the double-buffered binary Gibbs kernel):
    PCA and Gibbs sweeps interleaved one call at a time equal the oracle's sequence, and a
    checkpoint (state, counts, step) resumed in a fresh context continues the same chain."""
    H, W = 32, 64
    g = synth.degrade(synth.smooth_labels(H, W, 2, 3), 2, 0.5, 4)
    cfg = P.make_config(H, W, 2, periodic=True, sigma=0.5, beta0=1.2, beta_step=0.2,
                        beta_period=3, seed=13, mpm_burn_in=2)
    ctx = make_ctx(cfg, g)
    plan = ["pca", "gibbs", "gibbs", "pca", "gibbs", "pca", "gibbs"]
    for step in plan[:4]:
        (ctx.pca_sweep if step == "pca" else ctx.pca_gibbs_sweep)(1)
    # checkpoint after 4 sweeps
    x4, c4 = ctx.state(), ctx.counts()
    resumed = make_ctx(cfg, g, x4)
    resumed.pca_write_counts(c4, ctx.pca_get_stats().counted_sweeps)
    resumed.pca_set_step(4)
    for step in plan[4:]:
        for c in (ctx, resumed):
            (c.pca_sweep if step == "pca" else c.pca_gibbs_sweep)(1)
    assert np.array_equal(ctx.state(), resumed.state())
    assert np.array_equal(ctx.counts(), resumed.counts())
    m = oracle_model(cfg)
    x = g.copy()
    cnt = np.zeros((H, W), np.uint16)
    for t, step in enumerate(plan):
        beta = beta_of(cfg, t)
        x = orc.pca_sweep(m, x, g, beta, 13, 0, t)[0] if step == "pca" else \
            orc.gibbs_sweep_coloured(m, x, g, beta, 13, 0, t)
        if t >= 2:
            cnt += x
    assert np.array_equal(ctx.state()[0], x) and np.array_equal(ctx.counts()[0], cnt)
