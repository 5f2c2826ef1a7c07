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


def _cudart_copy():
    from test_gpu_parity import _cudart_memcpy
    return _cudart_memcpy()


def _strip_bounds(H):
    return [0, H // 3, (2 * H) // 3 + 1, H]


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("nbhd", [8, 4])
def test_row_strips_two_sweeps_per_pass_loopback(cuda_device, periodic, nbhd):
    """SURVEY 8(f) rank 1 on row strips: each strip context advances two sweeps per pass
    (recomputing sweep t one row beyond its edges from the 2-deep x halo and the g halo row),
    and the caller exchanges the 2-row halos once per pass -- half the messages of one sweep
    per pass.  The strips reproduce the oracle's unsharded chain and MPM counts bit for bit,
    across beta stages, the burn-in and an odd trailing sweep."""
    import torch

    copy = _cudart_copy()
    H, W, Pn = 45, 1040, 3
    g = synth.degrade(synth.smooth_labels(H, W, 2, 7), 2, 0.45, 8)
    base = dict(neighborhood=nbhd, periodic=periodic, sigma=0.45, beta0=1.0, beta_step=0.3,
                beta_period=3, seed=31, mpm_burn_in=3, sweeps_per_pass=2, kernel=P.KERNEL_BINARY)
    b = _strip_bounds(H)
    strips = [make_ctx(P.make_config(H, W, 2, row0=b[i], rows=b[i + 1] - b[i], **base), g[b[i]:b[i + 1]])
              for i in range(Pn)]

    def peers(i):
        up, dn = i - 1, i + 1
        if periodic:
            up, dn = up % Pn, dn % Pn
        return up, dn

    def exchange(g_rows=False):
        torch.cuda.synchronize()
        hs = [s.pca_halo_ptrs() for s in strips]
        for i in range(Pn):
            up, dn = peers(i)
            if 0 <= up < Pn:
                copy(hs[i].recv_top, hs[up].send_bottom, hs[i].row_bytes)
                if g_rows:
                    copy(hs[i].g_recv_top, hs[up].g_send_bottom, hs[i].g_row_bytes)
            if 0 <= dn < Pn:
                copy(hs[i].recv_bottom, hs[dn].send_top, hs[i].row_bytes)
                if g_rows:
                    copy(hs[i].g_recv_bottom, hs[dn].g_send_top, hs[i].g_row_bytes)
        torch.cuda.synchronize()

    exchange(g_rows=True)
    l0 = [s.pca_get_stats().sweep_launches for s in strips]
    for _ in range(5):          # 5 passes = 10 sweeps, one exchange per pass
        for s in strips:
            s.pca_sweep(2)
        exchange()
    for s in strips:            # an odd trailing sweep (2-deep halos again afterwards)
        s.pca_sweep(1)
    exchange()
    for s, l in zip(strips, l0):
        assert s.pca_get_stats().sweep_launches - l == 6  # 5 passes + 1 single sweep
    got = np.concatenate([s.state()[0] for s in strips], axis=0)
    gc = np.concatenate([s.counts()[0] for s in strips], axis=0)
    x_o, cnt_o = orc.pca_run(oracle_model(P.make_config(H, W, 2, **base)), g, g, 11, 1.0, 0.3, 3, 31,
                             burn_in=3)
    assert np.array_equal(got, x_o)
    assert np.array_equal(gc, cnt_o[1].astype(np.uint16))


@pytest.mark.parametrize("periodic", [True, False])
def test_row_strips_two_sweeps_per_pass_over_peers(cuda_device, periodic):
    """The same with attached peers (device-initiated halo path, one phase per pass: the pass
    kernel, then its 2 edge rows of x_{t+2} copied into the neighbours' halos; the g halo rows
    pushed once in the first pass), runs of several passes per call."""
    import torch

    from test_gpu_peers import _attach, _strips

    H, W = 48, 1040
    g = synth.degrade(synth.smooth_labels(H, W, 2, 9), 2, 0.45, 10)[None]
    base = dict(neighborhood=8, periodic=periodic, sigma=0.45, beta0=1.0, beta_step=0.3, beta_period=3,
                seed=41, mpm_burn_in=2, sweeps_per_pass=2, kernel=P.KERNEL_BINARY)
    # one stream per strip, as on separate GPUs: a call with several phases (the g push, then
    # the passes) waits on the neighbours' phases, which they issue after this call returns
    strips = _strips(H, W, 2, [0, 16, 31, 48], base, g, [torch.cuda.Stream() for _ in range(3)])
    _attach(strips, periodic)
    l0 = [s.pca_get_stats().sweep_launches for s in strips]
    for n in (2, 5, 4):
        for s in strips:
            s.pca_sweep(n)
    torch.cuda.synchronize()
    for s, l in zip(strips, l0):
        assert s.pca_get_stats().sweep_launches - l == 1 + 3 + 2  # passes (+ the odd sweep)
    got = np.concatenate([s.state() for s in strips], axis=1)[0]
    gc = np.concatenate([s.counts() for s in strips], axis=-2)[0]
    x_o, cnt_o = orc.pca_run(oracle_model(P.make_config(H, W, 2, **base)), g[0], g[0], 11, 1.0, 0.3, 3, 41,
                             burn_in=2)
    assert np.array_equal(got, x_o)
    assert np.array_equal(gc, cnt_o[1].astype(np.uint16))
    for s in strips:
        s.pca_destroy()
