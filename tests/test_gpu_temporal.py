"""-m gpu parity of the two-sweeps-per-pass binary kernel (sweep_binary2.cu, temporal
blocking): it must produce exactly the chain of two single sweeps -- vs the oracle in
pair-lockstep (the oracle advances two sweeps from the GPU's state) and vs the one-sweep
kernel (same context config with sweeps_per_pass = 1), including MPM counts across
burn-in and beta-stage boundaries that fall between the two sweeps of a pass."""
import numpy as np
import pytest

import oracle as orc
import paper_2507_14869_b200 as P
import synth
from parity_helpers import Tally, beta_of, make_ctx, oracle_model

pytestmark = pytest.mark.gpu

# W % 16 == 0 (the kernel's requirement); several 512-column segments, partial last segment,
# tiny lattices, single-segment lattices
SHAPES = [(64, 64), (37, 528), (3, 16), (5, 1040), (40, 1536), (130, 48), (16, 2064)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}x{s[1]}")
@pytest.mark.parametrize("nbhd", [4, 8])
@pytest.mark.parametrize("periodic", [True, False])
def test_pair_lockstep_vs_oracle(cuda_device, shape, nbhd, periodic):
    H, W = shape
    cfg = P.make_config(H, W, 2, neighborhood=nbhd, periodic=periodic, sigma=0.5, beta0=0.9,
                        beta_step=0.4, beta_period=3, seed=H * 7919 + W, mpm_burn_in=-1,
                        sweeps_per_pass=2)
    g = synth.random_labels((H, W), 2, seed=H + 3 * W)
    x0 = synth.random_labels((H, W), 2, seed=2 * H + W)
    ctx = make_ctx(cfg, g, x0)
    m = oracle_model(cfg)
    tally = Tally()
    x = ctx.state()[0]
    for t in range(0, 8, 2):
        ctx.pca_sweep(2)
        assert ctx.pca_get_stats().sweeps_done == t + 2
        x1, _ = orc.pca_sweep(m, x, g, beta_of(cfg, t), cfg.seed, 0, t)
        x2, mg = orc.pca_sweep(m, x1, g, beta_of(cfg, t + 1), cfg.seed, 0, t + 1)
        got = ctx.state()[0]
        tally.add(got, x2, mg)
        x = got
    tally.check(allow_rate=False)


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("nbhd", [4, 8])
def test_two_per_pass_equals_one_per_pass(cuda_device, periodic, nbhd):
    """Same chain and MPM counts as one sweep per launch, with the burn-in (counting starts
    at t = 7, mid-pass) and beta stages (period 5) falling between the two sweeps of a pass."""
    H, W = 96, 1024
    g = synth.degrade(synth.smooth_labels(H, W, 2, 4), 2, 0.5, 5)
    kw = dict(neighborhood=nbhd, periodic=periodic, sigma=0.5, beta0=1.1, beta_step=0.2,
              beta_period=5, seed=99, mpm_burn_in=7)
    a = make_ctx(P.make_config(H, W, 2, sweeps_per_pass=2, **kw), g)
    b = make_ctx(P.make_config(H, W, 2, sweeps_per_pass=1, **kw), g)
    for n in (3, 8, 1, 12):  # odd counts exercise the single-sweep tail
        a.pca_sweep(n)
        b.pca_sweep(n)
        assert np.array_equal(a.state(), b.state())
        assert np.array_equal(a.counts(), b.counts())
    sa, sb = a.pca_get_stats(), b.pca_get_stats()
    assert sa.sweeps_done == sb.sweeps_done == 24 and sa.counted_sweeps == sb.counted_sweeps == 17
    assert sa.sweep_launches == 2 + 4 + 1 + 6  # pairs + single-sweep tails


def test_two_per_pass_full_size_sampled_rows(cuda_device):
    """Config 3 size (8192^2, Moore-8 torus, MPM on): 2 sweeps in one pass, sampled rows
    recomputed by the oracle from the GPU's x_t through x_{t+1}."""
    H = W = 8192
    g = synth.degrade(synth.tiled_labels(H, W, 2, seed=1), 2, 0.5, seed=2)
    cfg = P.make_config(H, W, 2, neighborhood=8, periodic=True, sigma=0.5, beta0=1.5,
                        beta_step=0.0, seed=11, mpm_burn_in=0, sweeps_per_pass=2)
    ctx = make_ctx(cfg, g)
    ctx.pca_sweep(2)
    x2 = ctx.state()[0]
    ctx.pca_sweep(2)
    x4 = ctx.state()[0]
    m = oracle_model(cfg)
    rng = np.random.default_rng(0)
    rows = sorted({0, 1, H - 2, H - 1, H // 2} | set(rng.integers(2, H - 2, 20).tolist()))
    tally = Tally()
    for r in rows:
        lo, hi = r - 1, r + 2  # x3 rows r-1..r+1 needed for x4 row r
        span = [(q % H) for q in range(lo, hi)]
        x3_rows = {}
        for q in span:
            out, _ = orc.pca_sweep(m, x2, g, 1.5, cfg.seed, 0, 2, rows=(q, q + 1))
            x3_rows[q] = out[0]
        x3 = x2.copy()
        for q, v in x3_rows.items():
            x3[q] = v
        ref, mg = orc.pca_sweep(m, x3, g, 1.5, cfg.seed, 0, 3, rows=(r, r + 1))
        tally.add(x4[r], ref[0], mg[0])
    tally.check()
    assert ctx.counts()[0].max() <= 4
