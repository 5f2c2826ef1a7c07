"""-m gpu: the bit-packed two-level sweep (PCA_KERNEL_PACKED, sweep_packed.cu; north star (2),
SURVEY 2.3 K2) against the oracle and against the byte kernel.

The packed kernel draws the same Philox words and decides with the same integer thresholds as
the byte kernel, so the chains must be identical bit for bit (no near-tie exceptions exist on
the two-level integer path)."""
import numpy as np
import pytest

import oracle as orc
import paper_2507_14869_b200 as P
import synth
from parity_helpers import Tally, lockstep, make_ctx, oracle_model

pytestmark = pytest.mark.gpu

SHAPES = [(24, 512, 8, True), (33, 1024, 8, False), (40, 512, 4, True), (17, 1536, 4, False),
          (3, 512, 8, True), (5, 2048, 8, False)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_packed_lockstep_random_states(cuda_device, shape):
    H, W, nb, per = shape
    cfg = P.make_config(H, W, 2, neighborhood=nb, periodic=per, sigma=0.4, beta0=0.9, beta_step=0.5,
                        beta_period=2, seed=77 + H, mpm_burn_in=2, kernel=P.KERNEL_PACKED)
    g = synth.random_labels((H, W), 2, seed=H + W)
    x0 = synth.random_labels((H, W), 2, seed=H * W)
    ctx = make_ctx(cfg, g, x0)
    assert ctx.pca_get_stats().kernel == P.KERNEL_PACKED
    lockstep(ctx, cfg, 6).check(allow_rate=False)


@pytest.mark.parametrize("per", [True, False])
@pytest.mark.parametrize("nb", [8, 4])
def test_packed_runs_equal_byte_kernel_and_oracle(cuda_device, per, nb):
    """Runs of sweeps in one call (pack once, n packed sweeps, unpack x_t and x_{t-1}) across
    beta stages and the MPM burn-in, on a lattice above the multi-sweep threshold, equal the
    byte kernel (states, counts, changed sites) and the oracle's chain; batch of 2 chains."""
    H, W, B = 300, 1024, 2
    truth = np.stack([synth.smooth_labels(H, W, 2, seed=10 + b) for b in range(B)])
    g = np.stack([synth.degrade(truth[b], 2, 0.45, seed=20 + b) for b in range(B)])
    kw = dict(batch=B, neighborhood=nb, periodic=per, sigma=0.45, beta0=1.1, beta_step=0.2,
              beta_period=7, seed=5, mpm_burn_in=9)
    a = make_ctx(P.make_config(H, W, 2, kernel=P.KERNEL_PACKED, **kw), g)
    b = make_ctx(P.make_config(H, W, 2, kernel=P.KERNEL_BINARY, **kw), g)
    for n in (1, 5, 13, 2):
        for c in (a, b):
            c.pca_sweep(n)
        assert np.array_equal(a.state(), b.state())
        assert np.array_equal(a.counts(), b.counts())
        assert np.array_equal(a.pca_changed_sites(), b.pca_changed_sites())
    m = oracle_model(a.cfg)
    for ch in range(B):
        x_o, cnt_o = orc.pca_run(m, g[ch], g[ch], 21, 1.1, 0.2, 7, 5, chain=ch, burn_in=9)
        assert np.array_equal(a.state()[ch], x_o)
        assert np.array_equal(a.counts()[ch], cnt_o[1].astype(np.uint16))
    pa, sa = a.pca_finalize(truth, np.zeros_like(truth))
    pb, sb = b.pca_finalize(truth, np.zeros_like(truth))
    assert np.array_equal(pa, pb) and np.array_equal(sa, sb)
    # a reset with a new g repacks g; Gibbs sweeps in between use the byte state
    g2 = np.ascontiguousarray(g[::-1])
    for c in (a, b):
        c.pca_reset(g2, None)
        c.pca_sweep(3)
        c.pca_gibbs_sweep(1)
        c.pca_sweep(4)
    assert np.array_equal(a.state(), b.state())
    assert np.array_equal(a.counts(), b.counts())


def test_packed_full_size_8192(cuda_device):
    """Config 3 (8192^2, Moore-8 torus, MPM on) on the packed kernel: three sweeps in one call
    and one more equal the byte kernel bit for bit, and sampled rows of the last sweep are
    recomputed by the oracle from the GPU's x_t."""
    H = W = 8192
    truth = synth.tiled_labels(H, W, 2, seed=1)
    g = synth.degrade(truth, 2, 0.5, seed=2)
    kw = dict(neighborhood=8, periodic=True, sigma=0.5, beta0=1.5, beta_step=0.0, seed=11, mpm_burn_in=0)
    a = make_ctx(P.make_config(H, W, 2, kernel=P.KERNEL_PACKED, **kw), g)
    a.pca_sweep(3)
    x3 = a.state()[0]
    a.pca_sweep(1)
    x4 = a.state()[0]
    b = make_ctx(P.make_config(H, W, 2, kernel=P.KERNEL_BINARY, **kw), g)
    b.pca_sweep(4)
    assert np.array_equal(x4, b.state()[0])
    assert np.array_equal(a.counts(), b.counts())
    m = oracle_model(a.cfg)
    tally = Tally()
    rows = sorted({0, 1, H - 2, H - 1, H // 2} | set(np.random.default_rng(4).integers(0, H, 24).tolist()))
    for r in rows:
        ref, mg = orc.pca_sweep(m, x3, g, 1.5, 11, 0, 3, rows=(r, r + 1))
        tally.add(x4[r], ref[0], mg[0])
    tally.check(allow_rate=False)


def test_packed_kernel_rejects_ineligible_configs(cuda_device):
    for kw in (dict(height=64, width=500, levels=2), dict(height=64, width=512, levels=3),
               dict(height=2, width=512, levels=2)):
        with pytest.raises(P.PcaError):
            P.pca_workspace_bytes(P.make_config(kw.pop("height"), kw.pop("width"), kw.pop("levels"),
                                                kernel=P.KERNEL_PACKED, **kw))


def test_packed_count_deltas_fold_across_long_runs(cuda_device):
    """The packed kernel's uint8 count deltas are folded into the uint16 counts every 255
    counted sweeps and at the end of each call: 600 counted sweeps in one call, then 300 in
    another, equal the byte kernel's counts (and the MPM image)."""
    H, W = 260, 1024
    g = synth.degrade(synth.smooth_labels(H, W, 2, seed=3), 2, 0.45, seed=4)
    kw = dict(neighborhood=8, periodic=True, sigma=0.45, beta0=1.2, beta_step=0.0, seed=8, mpm_burn_in=3)
    a = make_ctx(P.make_config(H, W, 2, kernel=P.KERNEL_PACKED, **kw), g)
    b = make_ctx(P.make_config(H, W, 2, kernel=P.KERNEL_BINARY, **kw), g)
    for n in (603, 300):
        for c in (a, b):
            c.pca_sweep(n)
        assert np.array_equal(a.state(), b.state())
        assert np.array_equal(a.counts(), b.counts())
    assert a.pca_get_stats().counted_sweeps == 900
    assert np.array_equal(a.estimate(P.EST_MPM), b.estimate(P.EST_MPM))


def _loopback_exchange(strips, periodic):
    """Copy every strip's 2-row edges into its neighbours' halo rows, chain by chain (the caller's
    exchange of a strip context without NCCL or peers, pca_halo_ptrs)."""
    import torch

    from test_gpu_parity import _cudart_memcpy

    copy = _cudart_memcpy()
    torch.cuda.synchronize()
    hs = [s.pca_halo_ptrs() for s in strips]
    n = len(strips)
    for b in range(strips[0].cfg.batch):
        for i in range(n):
            up, dn = i - 1, i + 1
            if periodic:
                up, dn = up % n, dn % n
            o = b * hs[i].chain_stride
            if 0 <= up < n:
                copy(hs[i].recv_top + o, hs[up].send_bottom + b * hs[up].chain_stride, hs[i].row_bytes)
            if 0 <= dn < n:
                copy(hs[i].recv_bottom + o, hs[dn].send_top + b * hs[dn].chain_stride, hs[i].row_bytes)
    torch.cuda.synchronize()


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("nb", [8, 4])
def test_packed_row_strips_loopback(cuda_device, periodic, nb):
    """Row strips on the packed kernel: each sweep is the strip's edge rows and its
    interior as separate row ranges of the packed kernel, unpacked with the neighbours' halo rows;
    strips of 2 rows (one launch), 3 rows and more, batch of 2 chains, exchanged by the caller
    after every sweep, reproduce the unsharded packed chain and the oracle's chain bit for bit."""
    H, W, B = 64, 1024, 2
    truth = np.stack([synth.smooth_labels(H, W, 2, seed=30 + b) for b in range(B)])
    g = np.stack([synth.degrade(truth[b], 2, 0.4, seed=40 + b) for b in range(B)])
    base = dict(batch=B, neighborhood=nb, periodic=periodic, sigma=0.4, seed=13, mpm_burn_in=3,
                beta_period=4, kernel=P.KERNEL_PACKED)
    full = make_ctx(P.make_config(H, W, 2, **base), g)
    bounds = [0, 2, 5, 26, 64]
    strips = [make_ctx(P.make_config(H, W, 2, row0=bounds[i], rows=bounds[i + 1] - bounds[i], **base),
                       np.ascontiguousarray(g[:, bounds[i]:bounds[i + 1]])) for i in range(len(bounds) - 1)]
    for s in strips:
        assert s.pca_get_stats().kernel == P.KERNEL_PACKED
    _loopback_exchange(strips, periodic)
    n = 9
    for _ in range(n):
        for s in strips:
            s.pca_sweep(1)
        _loopback_exchange(strips, periodic)
    full.pca_sweep(n)
    got = np.concatenate([s.state() for s in strips], axis=1)
    assert np.array_equal(got, full.state())
    gc = np.concatenate([s.counts() for s in strips], axis=-2)
    assert np.array_equal(gc, full.counts())
    for ch in range(B):
        x_o, cnt_o = orc.pca_run(oracle_model(full.cfg), g[ch], g[ch], n, 1.25, 0.25, 4, 13, chain=ch,
                                 burn_in=3)
        assert np.array_equal(got[ch], x_o)
        assert np.array_equal(gc[ch], cnt_o[1].astype(np.uint16))
    # 3 launches per sweep on strips of >= 3 rows (edges, interior), 1 on the 2-row strip
    assert strips[0].pca_get_stats().sweep_launches == n
    assert strips[1].pca_get_stats().sweep_launches == 3 * n
    for s in strips:
        s.pca_destroy()


@pytest.mark.parametrize("periodic", [True, False])
def test_packed_strips_attached_to_peers_run_the_byte_kernel(cuda_device, periodic):
    """A packed-eligible strip with device-initiated peers sweeps the byte state with the binary
    kernel (the peer stores live there): still the unsharded chain bit for bit."""
    import torch

    from test_gpu_peers import _attach, _strips

    H, W = 40, 512
    g = synth.degrade(synth.smooth_labels(H, W, 2, 3), 2, 0.4, 4)[None]
    base = dict(neighborhood=8, periodic=periodic, sigma=0.4, seed=21, mpm_burn_in=2)
    full = P.PcaContext(P.make_config(H, W, 2, **base), g)
    strips = _strips(H, W, 2, [0, 13, 40], base, g, torch.cuda.Stream())
    assert strips[0].pca_get_stats().kernel == P.KERNEL_PACKED
    _attach(strips, periodic)
    for _ in range(7):
        for s in strips:
            s.pca_sweep(1)
    full.pca_sweep(7)
    assert np.array_equal(np.concatenate([s.state() for s in strips], axis=1), full.state())
    assert np.array_equal(np.concatenate([s.counts() for s in strips], axis=-2), full.counts())
    for s in strips:
        s.pca_destroy()
