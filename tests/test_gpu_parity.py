"""-m gpu parity: the CUDA path (through the C ABI) vs the fp64 CPU oracle.

Bar (BASELINE.json north star, R19): chains bit-exact; the only allowed differences are
decision mismatches whose uniform lies within 1e-6 of an oracle cumulative probability,
fewer than 1e-6 of all updates.  Integer outputs (MPM counts, MPM image) exact; PSNR within
0.01 dB and SSIM within 1e-9 of the oracle's two-pass fp64 statistics.
"""
import math

import numpy as np
import pytest

import oracle as orc
import paper_2507_14869_b200 as P
import synth
from parity_helpers import Tally, beta_of, lockstep, make_ctx, oracle_model

pytestmark = pytest.mark.gpu


# (H, W, levels, nbhd, periodic): several tiles, ragged widths (not multiples of 16 / 4),
# single rows / columns, and the paper's level counts.
SHAPES = [
    (64, 64, 2, 4, True), (64, 64, 2, 8, False), (37, 531, 2, 8, True), (19, 1000, 2, 4, False),
    (1, 77, 2, 8, False), (77, 1, 2, 8, False), (3, 3, 2, 8, True), (5, 17, 2, 8, False),
    (33, 47, 3, 8, False), (40, 130, 5, 8, False), (29, 61, 9, 4, True), (31, 45, 33, 8, False),
    (9, 23, 255, 8, True), (2, 2, 3, 8, False), (1, 1, 5, 8, False),
    # W % 16 == 0 with 3, 5, 9 levels: the general sweep's TMA path (several segments, ragged)
    (21, 48, 3, 8, True), (37, 1040, 5, 8, False), (30, 64, 9, 4, True), (5, 16, 5, 8, False),
    # the compile-time level counts with 4 neighbours (shared-memory W0 weights, SWAR table
    # rows) and 16 levels (the largest fixed path)
    (26, 70, 5, 4, False), (20, 36, 3, 4, True), (23, 50, 16, 8, True), (18, 41, 16, 4, False),
    # 4 levels (the table kernel's middle instantiation; the general kernel's run-time path)
    (27, 61, 4, 8, True), (19, 130, 4, 4, False),
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("kernel", [P.KERNEL_AUTO, P.KERNEL_GENERAL])
def test_lockstep_random_states(cuda_device, shape, kernel):
    H, W, L, nb, per = shape
    cfg = P.make_config(H, W, L, neighborhood=nb, periodic=per, sigma=0.3, beta0=0.9,
                        beta_step=0.5, beta_period=2, seed=1234 + H * W, kernel=kernel)
    g = synth.random_labels((H, W), L, seed=H * 1000 + W)
    x0 = synth.random_labels((H, W), L, seed=W * 1000 + H)
    ctx = make_ctx(cfg, g, x0)
    tally = lockstep(ctx, cfg, 6)
    tally.check(allow_rate=False)


@pytest.mark.parametrize("levels", [3, 4, 5])
@pytest.mark.parametrize("nb,periodic,W", [(8, False, 257), (8, True, 96), (4, True, 130), (4, False, 64)])
def test_table_kernel_lockstep_and_agreement(cuda_device, levels, nb, periodic, W):
    """The histogram-table kernel (3..5 levels, AUTO's choice): smooth states with sprinkled
    random labels exercise both the table rows (<= 2 neighbour labels) and the queued fp64
    sites; lockstep against the oracle with zero mismatches, then 40 free-running sweeps with
    MPM counts equal to the general kernel's (PCA_KERNEL_GENERAL), including the multi-sweep
    launches of small contexts."""
    H = 70
    truth = synth.smooth_labels(H, W, levels, seed=levels * 10 + nb)
    g = synth.degrade(truth, levels, 0.3, seed=5)
    x0 = synth.smooth_labels(H, W, levels, seed=77)
    x0[::5, ::3] = synth.random_labels(x0[::5, ::3].shape, levels, seed=78)
    kw = dict(neighborhood=nb, periodic=periodic, sigma=0.3, beta0=1.1, beta_step=0.3,
              beta_period=3, seed=314 + levels, mpm_burn_in=5)
    cfg = P.make_config(H, W, levels, **kw)
    ctx = make_ctx(cfg, g, x0)
    assert ctx.pca_get_stats().kernel == P.KERNEL_TABLE
    lockstep(ctx, cfg, 6).check(allow_rate=False)
    a = make_ctx(cfg, g, x0)
    b = make_ctx(P.make_config(H, W, levels, kernel=P.KERNEL_GENERAL, **kw), g, x0)
    assert b.pca_get_stats().kernel == P.KERNEL_GENERAL
    for c in (a, b):
        c.pca_sweep(40)
    assert np.array_equal(a.state(), b.state())
    assert np.array_equal(a.counts(), b.counts())
    x_o, cnt_o = orc.pca_run(oracle_model(cfg), x0, g, 40, 1.1, 0.3, 3, cfg.seed, burn_in=5)
    assert np.array_equal(a.state()[0], x_o)
    assert np.array_equal(a.counts()[0], cnt_o.astype(np.uint16))


@pytest.mark.parametrize("levels,nb,periodic", [(5, 8, False), (3, 4, True), (4, 8, True)])
def test_table_kernel_count_deltas_fold_across_long_runs(cuda_device, levels, nb, periodic):
    """The table kernel's uint8 count deltas (one plane per level) are folded into the uint16
    counts before 255 counted sweeps accumulate and at the end of every call: 600 counted
    sweeps in one call, 300 in another, then single sweeps, on a context above the multi-sweep
    threshold with a ragged width (W % 16 != 0: the fold covers the last partial chunk), equal
    the general kernel's uint16 counts, and every estimate that reads them agrees."""
    H, W, B = 300, 517, 2
    truth = np.stack([synth.smooth_labels(H, W, levels, seed=40 + b) for b in range(B)])
    g = np.stack([synth.degrade(truth[b], levels, 0.3, seed=50 + b) for b in range(B)])
    kw = dict(batch=B, neighborhood=nb, periodic=periodic, sigma=0.3, beta0=1.3, beta_step=0.0, seed=9,
              mpm_burn_in=0)
    a = make_ctx(P.make_config(H, W, levels, **kw), g)
    b = make_ctx(P.make_config(H, W, levels, kernel=P.KERNEL_GENERAL, **kw), g)
    assert a.pca_get_stats().kernel == P.KERNEL_TABLE
    for n in (600, 300, 1, 1, 1):
        for c in (a, b):
            c.pca_sweep(n)
        assert np.array_equal(a.state(), b.state())
        assert np.array_equal(a.counts(), b.counts())
    assert a.pca_get_stats().counted_sweeps == 903
    for est in (P.EST_MPM, P.EST_CM):
        assert np.array_equal(a.estimate(est), b.estimate(est))
    pa, sa = a.pca_finalize(truth, np.zeros_like(truth))
    pb, sb = b.pca_finalize(truth, np.zeros_like(truth))
    assert np.array_equal(pa, pb) and np.array_equal(sa, sb)


@pytest.mark.parametrize("levels,W,kernel,graphs", [(2, 512, P.KERNEL_PACKED, 1), (2, 512, P.KERNEL_PACKED, 0),
                                                   (5, 517, P.KERNEL_TABLE, 0), (2, 520, P.KERNEL_BINARY, 1)])
def test_run_refused_at_the_counter_limit_keeps_a_consistent_state(cuda_device, levels, W, kernel, graphs):
    """A run refused part-way (the 65535th counted sweep is the last a uint16 counter holds)
    executes the sweeps before the refusal and leaves state, sweep index and counts consistent
    with them -- on the packed kernel (its state is unpacked, its deltas folded), the table
    kernel (deltas folded) and the byte kernel, with and without graph capture."""
    H = 520  # above the multi-sweep threshold, so the per-kernel paths run
    g = synth.degrade(synth.smooth_labels(H, W, levels, 3), levels, 0.4, 4)
    kw = dict(neighborhood=8, periodic=True, sigma=0.4, seed=6, mpm_burn_in=0, kernel=kernel,
              graphs=graphs if levels == 2 else 0)
    a = make_ctx(P.make_config(H, W, levels, **kw), g)
    ref = make_ctx(P.make_config(H, W, levels, **kw), g)
    assert a.pca_get_stats().kernel == kernel
    c0 = a.counts()
    a.pca_write_counts(c0, 65530)
    with pytest.raises(P.PcaError, match="65535"):
        a.pca_sweep(12)
    st = a.pca_get_stats()
    assert st.sweeps_done == 5 and st.counted_sweeps == 65535
    ref.pca_sweep(5)
    assert np.array_equal(a.state(), ref.state())
    assert np.array_equal(a.counts(), ref.counts())
    assert np.array_equal(a.pca_changed_sites(), ref.pca_changed_sites())
    with pytest.raises(P.PcaError, match="65535"):  # nothing left to count into
        a.pca_sweep(1)
    assert a.pca_get_stats().sweeps_done == 5
    assert np.array_equal(a.state(), ref.state())


@pytest.mark.parametrize("q", [0.0, 0.51, 3.0, 1e6])
def test_lockstep_inertia_extremes(cuda_device, q):
    cfg = P.make_config(48, 80, 2, neighborhood=8, periodic=False, q=q, sigma=0.5, seed=7)
    g = synth.smooth_labels(48, 80, 2, seed=3)
    ctx = make_ctx(cfg, synth.degrade(g, 2, 0.5, 4))
    lockstep(ctx, cfg, 5).check(allow_rate=False)
    if q == 1e6:  # infinite inertia freezes the chain
        assert np.array_equal(ctx.state()[0], ctx._g_host[0])


@pytest.mark.parametrize("inertia_p", [1, 2])
@pytest.mark.parametrize("shape", [(40, 130, 5, 8, False), (29, 61, 9, 4, True),
                                   (31, 45, 33, 8, False), (33, 47, 2, 8, True),
                                   (24, 528, 5, 8, True), (18, 64, 9, 8, False)],
                         ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("q", [0.51, 4.0, 1e6])
def test_lockstep_l1_l2_inertia(cuda_device, inertia_p, shape, q):
    """L1 / L2 inertia norms, table (levels <= 16) and fp64 paths,
    including the log-domain path (q = 1e6 under/overflows the factorised weights)."""
    H, W, L, nb, per = shape
    cfg = P.make_config(H, W, L, neighborhood=nb, periodic=per, q=q, sigma=0.3, beta0=0.9,
                        beta_step=0.5, beta_period=2, seed=99 + L, inertia_p=inertia_p)
    g = synth.smooth_labels(H, W, L, seed=5)
    x0 = synth.smooth_labels(H, W, L, seed=6)  # smooth: the uniform-table path is exercised
    x0[::3, ::2] = synth.random_labels(x0[::3, ::2].shape, L, seed=7)  # ... and the fp64 one
    ctx = make_ctx(cfg, synth.degrade(g, L, 0.3, 8), x0)
    lockstep(ctx, cfg, 6).check(allow_rate=False)


def _c1_config(seed, kernel=P.KERNEL_AUTO):
    # config 1 (BASELINE.json configs[0]): 64x64 binary, 4-neighbour torus, 200 sweeps,
    # schedule 1.25 + 0.25 every 50 (the paper's compressed), MPM burn-in 100.
    return P.make_config(64, 64, 2, neighborhood=4, periodic=True, sigma=0.5, beta0=1.25,
                         beta_step=0.25, beta_period=50, seed=seed, mpm_burn_in=100,
                         kernel=kernel)


def _c1_inputs(seed):
    m = orc.model(64, 64, 2, nbhd=4, periodic=True)
    truth = orc.generate_mrf(m, 400, 0.9, 1.6, seed=seed)
    return truth, orc.degrade(truth, 2, 0.5, seed=seed + 100)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_config1_free_running_chain(cuda_device, seed):
    """Free-running: GPU and oracle chains run independently for 200 sweeps; states,
    MPM counts, MPM image and PSNR/SSIM must agree exactly."""
    truth, g = _c1_inputs(seed)
    cfg = _c1_config(seed)
    ctx = make_ctx(cfg, g)
    ctx.pca_sweep(200)
    m = oracle_model(cfg)
    x_o, cnt_o = orc.pca_run(m, g, g, 200, 1.25, 0.25, 50, seed, burn_in=100)
    assert np.array_equal(ctx.state()[0], x_o)
    assert np.array_equal(ctx.counts()[0], cnt_o[1].astype(np.uint16))
    mpm_o = orc.mpm(cnt_o)
    assert np.array_equal(ctx.estimate(P.EST_MPM)[0], mpm_o)
    for kind, est in [(P.EST_LAST, x_o), (P.EST_MPM, mpm_o)]:
        psnr, ssim = ctx.pca_psnr_ssim(truth[None], kind)
        _, p_o, s_o, _ = orc.metrics(truth, est, 2)
        assert abs(psnr[0] - p_o) < 0.01 and abs(psnr[0] - p_o) < 1e-9
        assert abs(ssim[0] - s_o) < 1e-9
        sw = ctx.pca_ssim_windowed(truth[None], kind)
        assert abs(sw[0] - orc.ssim_windowed(truth, est, 2)) < 1e-12
    # the fused finalisation pass: MPM image + LAST and MPM metrics, host and device outputs
    for out in (np.zeros((1, 64, 64), np.uint8), _to_device(np.zeros((1, 64, 64), np.uint8))):
        pf, sf = ctx.pca_finalize(truth[None], out)
        got = out if isinstance(out, np.ndarray) else out.cpu().numpy()
        assert np.array_equal(got[0], mpm_o)
        for e, est in enumerate((x_o, mpm_o)):
            _, p_o, s_o, _ = orc.metrics(truth, est, 2)
            assert abs(pf[0, e] - p_o) < 1e-9 and abs(sf[0, e] - s_o) < 1e-9
    # a staged truth (copy stream, overlapping) gives the same result
    with pytest.raises(P.PcaError, match="staged"):
        ctx.pca_finalize(None)
    ctx.pca_stage_truth(truth[None].copy())
    ps, ss = ctx.pca_finalize(None)
    assert np.array_equal(ps, pf) and np.array_equal(ss, sf)
    marg = ctx.estimate(P.EST_MARGINALS)[0]
    assert np.allclose(marg[1], cnt_o[1] / 100.0, atol=1e-6)
    assert np.allclose(marg[0] + marg[1], 1.0, atol=1e-6)
    st = ctx.pca_get_stats()
    assert st.sweeps_done == 200 and st.counted_sweeps == 100 and st.kernel == P.KERNEL_BINARY


def test_config1_binary_and_general_kernels_agree(cuda_device):
    truth, g = _c1_inputs(9)
    a = make_ctx(_c1_config(9, P.KERNEL_BINARY), g)
    b = make_ctx(_c1_config(9, P.KERNEL_GENERAL), g)
    a.pca_sweep(200)
    b.pca_sweep(200)
    assert np.array_equal(a.state(), b.state())
    assert np.array_equal(a.counts(), b.counts())


@pytest.mark.parametrize("levels,sigma,ramp,n", [(5, 0.25, (0.8, 1.5), 1000),
                                                  (9, 0.20, (0.8, 1.85), 300),
                                                  (33, 0.10, (1.0, 3.0), 120)])
def test_config2_paper_protocol_lockstep(cuda_device, levels, sigma, ramp, n):
    """Config 2: 256x256, Moore-8, free boundary, beta 1.25 + 0.25 every
    250 sweeps, q = 0.51, x0 = g; lockstep vs the oracle (l = 5 for the full 1000 sweeps;
    l = 9, 33 for a prefix to bound the oracle's time), then MPM / PSNR / SSIM exact."""
    m = orc.model(256, 256, levels, nbhd=8, periodic=False)
    truth = orc.generate_mrf(m, 150, ramp[0], ramp[1], seed=levels)
    g = orc.degrade(truth, levels, sigma, seed=levels + 50)
    burn = max(0, n - 250)
    cfg = P.make_config(256, 256, levels, neighborhood=8, periodic=False, sigma=sigma,
                        seed=2025 + levels, mpm_burn_in=burn)
    ctx = make_ctx(cfg, g)
    tally = lockstep(ctx, cfg, n, count_from=burn)
    tally.check()
    # Estimates are compared in every case, never skipped: against the oracle's count rule
    # and metrics applied to the lockstep states (the GPU chain, each sweep of which the
    # oracle confirmed up to allowed near-ties), and -- when no near-tie occurred -- also
    # against the free-running oracle chain, which is then the same chain.
    x_g = ctx.state()[0]
    cnt_l = tally.counts[0]
    assert np.array_equal(ctx.counts()[0], cnt_l.astype(np.uint16))
    x_o, cnt_o = orc.pca_run(oracle_model(cfg), g, g, n, 1.25, 0.25, 250, cfg.seed, burn_in=burn)
    refs = [(x_g, cnt_l)]
    if tally.mismatches == 0:
        assert np.array_equal(x_g, x_o)
        assert np.array_equal(cnt_l, cnt_o)
        refs.append((x_o, cnt_o))
    for last, cnt in refs:
        for kind, est in [(P.EST_LAST, last), (P.EST_MPM, orc.mpm(cnt))]:
            psnr, ssim = ctx.pca_psnr_ssim(truth[None], kind)
            _, p_o, s_o, _ = orc.metrics(truth, est, levels)
            assert abs(psnr[0] - p_o) < 1e-9 and abs(ssim[0] - s_o) < 1e-9
            sw = ctx.pca_ssim_windowed(truth[None], kind)
            assert abs(sw[0] - orc.ssim_windowed(truth, est, levels)) < 1e-12
        assert np.array_equal(ctx.estimate(P.EST_MPM)[0], orc.mpm(cnt))
        cm = ctx.estimate(P.EST_CM)[0]
        ref = (np.arange(levels)[:, None, None] / (levels - 1) * cnt).sum(0) / (n - burn)
        assert np.allclose(cm, ref, atol=1e-6)
    # the north star's end-to-end tolerances against the FREE-RUNNING oracle chain hold in
    # every case: MPM marginals within 1e-3, PSNR within 0.01 dB
    marg = ctx.estimate(P.EST_MARGINALS)[0]
    if tally.mismatches == 0:
        assert np.abs(marg - cnt_o / (n - burn)).max() < 1e-3
    for kind, est in [(P.EST_LAST, x_o), (P.EST_MPM, orc.mpm(cnt_o))]:
        psnr, _ = ctx.pca_psnr_ssim(truth[None], kind)
        assert abs(psnr[0] - orc.metrics(truth, est, levels)[1]) < 0.01


@pytest.mark.parametrize("H,W,L", [(7, 7, 2), (8, 300, 5), (130, 9, 9), (71, 133, 255), (64, 64, 33)])
def test_windowed_ssim_matches_oracle(cuda_device, H, W, L):
    """pca_ssim_windowed (7x7 windows, sample moments, R16) == orc_ssim_windowed for LAST and
    MPM, per chain of a batch, with ragged widths and heights that span several blocks."""
    B = 3
    truth = np.stack([synth.smooth_labels(H, W, L, seed=11 + b) for b in range(B)])
    g = np.stack([synth.degrade(truth[b], L, 0.3, seed=b) for b in range(B)])
    cfg = P.make_config(H, W, L, batch=B, sigma=0.3, seed=5, mpm_burn_in=2)
    ctx = make_ctx(cfg, g)
    ctx.pca_sweep(6)
    for kind in (P.EST_LAST, P.EST_MPM):
        est = ctx.estimate(kind)
        for t_arg in (truth, _to_device(truth)):
            sw = ctx.pca_ssim_windowed(t_arg, kind)
            for b in range(B):
                assert abs(sw[b] - orc.ssim_windowed(truth[b], est[b], L)) < 1e-12
    assert abs(ctx.pca_ssim_windowed(ctx.state(), P.EST_LAST)[0] - 1.0) < 1e-14
    small = make_ctx(P.make_config(6, 40, 2, sigma=0.5), np.zeros((6, 40), np.uint8))
    with pytest.raises(P.PcaError):
        small.pca_ssim_windowed(np.zeros((1, 6, 40), np.uint8), P.EST_LAST)


def _to_device(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_batch_equals_independent_chains(cuda_device):
    """Batch mode: chain b of a batch == a single-chain context with chain0 = b."""
    B, H, W = 4, 40, 72
    g = np.stack([synth.degrade(synth.smooth_labels(H, W, 5, s), 5, 0.25, s + 9) for s in range(B)])
    cfg = P.make_config(H, W, 5, batch=B, sigma=0.25, seed=77, mpm_burn_in=10)
    ctx = make_ctx(cfg, g)
    ctx.pca_sweep(25)
    xs, cs = ctx.state(), ctx.counts()
    for b in range(B):
        c1 = P.make_config(H, W, 5, batch=1, sigma=0.25, seed=77, mpm_burn_in=10, chain0=b)
        one = make_ctx(c1, g[b])
        one.pca_sweep(25)
        assert np.array_equal(one.state()[0], xs[b])
        assert np.array_equal(one.counts()[0], cs[b])
    t = lockstep(make_ctx(cfg, g), cfg, 3)
    t.check(allow_rate=False)


def _cudart_memcpy():
    """cudaMemcpy (device to device) from the CUDA runtime torch loaded (test plumbing)."""
    import ctypes
    import glob
    import os

    import nvidia.cuda_runtime as cr

    path = sorted(glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*")))[0]
    rt = ctypes.CDLL(path)
    rt.cudaMemcpy.restype = ctypes.c_int
    rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]

    def copy(dst, src, n):
        assert rt.cudaMemcpy(dst, src, n, 3) == 0  # cudaMemcpyDeviceToDevice

    return copy


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("levels", [2, 5])
def test_row_strips_with_loopback_halo_exchange(cuda_device, periodic, levels):
    """Row-strip decomposition: P strip contexts on one GPU whose halo rows
    are copied between them after every sweep reproduce the unsharded chain bit-exactly."""
    import torch

    memcpy_d2d = _cudart_memcpy()

    H, W, Pn = 48, 100, 3
    g = synth.degrade(synth.smooth_labels(H, W, levels, 5), levels, 0.3, 6)
    base = dict(neighborhood=8, periodic=periodic, sigma=0.3, seed=99, mpm_burn_in=4)
    full = make_ctx(P.make_config(H, W, levels, **base), g)
    bounds = [0, 17, 30, 48]
    strips = [make_ctx(P.make_config(H, W, levels, row0=bounds[i], rows=bounds[i + 1] - bounds[i],
                                     **base), g[bounds[i]:bounds[i + 1]]) for i in range(Pn)]

    def exchange():
        torch.cuda.synchronize()
        hs = [s.pca_halo_ptrs() for s in strips]
        rb = hs[0].row_bytes
        for i in range(Pn):
            up, dn = i - 1, i + 1
            if periodic:
                up %= Pn
                dn %= Pn
            if 0 <= up < Pn:
                memcpy_d2d(hs[i].recv_top, hs[up].send_bottom, rb)
            if 0 <= dn < Pn:
                memcpy_d2d(hs[i].recv_bottom, hs[dn].send_top, rb)
        torch.cuda.synchronize()

    exchange()
    for _ in range(10):
        for s in strips:
            s.pca_sweep(1)
        exchange()
    full.pca_sweep(10)
    got = np.concatenate([s.state()[0] for s in strips], axis=0)
    assert np.array_equal(got, full.state()[0])
    gc = np.concatenate([s.counts()[0] for s in strips], axis=-2)
    assert np.array_equal(gc, full.counts()[0])
    # and against the oracle's unsharded chain (not only the GPU's own)
    x_o, cnt_o = orc.pca_run(oracle_model(full.cfg), g, g, 10, 1.25, 0.25, 250, 99, burn_in=4)
    assert np.array_equal(got, x_o)
    assert np.array_equal(gc, (cnt_o[1] if levels == 2 else cnt_o).astype(np.uint16))
    truth = synth.smooth_labels(H, W, levels, 5)
    tot = sum(s.pca_metric_sums(truth[bounds[i]:bounds[i + 1]][None], P.EST_LAST)
              for i, s in enumerate(strips))
    ref = full.pca_metric_sums(truth[None], P.EST_LAST)
    assert np.array_equal(tot[:, [0, 1, 2, 3, 4, 5, 7]], ref[:, [0, 1, 2, 3, 4, 5, 7]])
    with pytest.raises(P.PcaError, match="row strip"):  # windows would span ranks
        strips[0].pca_ssim_windowed(truth[bounds[0]:bounds[1]][None], P.EST_LAST)


def test_checkpoint_resume_is_bit_exact(cuda_device):
    H, W = 50, 70
    g = synth.degrade(synth.smooth_labels(H, W, 2, 8), 2, 0.5, 9)
    cfg = P.make_config(H, W, 2, sigma=0.5, seed=5, mpm_burn_in=20, beta_period=15)
    a = make_ctx(cfg, g)
    a.pca_sweep(60)
    b = make_ctx(cfg, g)
    b.pca_sweep(35)
    st, cnt, t = b.state(), b.counts(), b.pca_get_stats()
    c = make_ctx(cfg, g)
    c.pca_write_state(st)
    c.pca_write_counts(cnt, t.counted_sweeps)
    c.pca_set_step(t.sweeps_done)
    c.pca_sweep(25)
    assert np.array_equal(c.state(), a.state()) and np.array_equal(c.counts(), a.counts())


def test_device_and_host_buffers_agree(cuda_device):
    import torch

    H, W = 33, 90
    g = synth.random_labels((1, H, W), 3, 4)
    cfg = P.make_config(H, W, 3, sigma=0.4, seed=3, mpm_burn_in=0)
    a = make_ctx(cfg, g)
    b = P.PcaContext(cfg, torch.from_numpy(g).cuda())
    a.pca_sweep(7)
    b.pca_sweep(7)
    out = torch.empty((1, H, W), dtype=torch.uint8, device="cuda")
    b.pca_estimate(P.EST_MPM, out)
    assert np.array_equal(out.cpu().numpy(), a.estimate(P.EST_MPM))
    assert np.array_equal(b.state(), a.state())


def test_error_paths(cuda_device):
    H, W = 16, 16
    g = synth.random_labels((H, W), 2, 1)
    bad = g.copy()
    bad[3, 3] = 7
    with pytest.raises(P.PcaError) as e:
        make_ctx(P.make_config(H, W, 2), bad)
    assert e.value.status == P.PCA_EINVAL
    ctx = make_ctx(P.make_config(H, W, 2, mpm_burn_in=-1), g)
    with pytest.raises(P.PcaError):
        ctx.estimate(P.EST_MPM)
    ctx.pca_sweep(0)
    assert np.array_equal(ctx.state()[0], g)  # zero sweeps: final = initial
    with pytest.raises(P.PcaError) as e:
        ctx.pca_write_state(bad)
    assert e.value.status == P.PCA_EINVAL
    # a failed load leaves labels >= levels in the buffer: calls that read the state refuse
    # until a valid load, and a valid one makes the context usable again
    for call in (lambda: ctx.pca_sweep(1), ctx.state, lambda: ctx.pca_gibbs_sweep(1)):
        with pytest.raises(P.PcaError) as e:
            call()
        assert e.value.status == P.PCA_ESTATE
    ctx.pca_write_state(g)
    # the same for a failed reset with a new g on a context that has swept (the fused reset
    # writes x[0] in the pass that checks g)
    ctx.pca_sweep(2)
    with pytest.raises(P.PcaError) as e:
        ctx.pca_reset(bad, None)
    assert e.value.status == P.PCA_EINVAL
    with pytest.raises(P.PcaError) as e:
        ctx.pca_sweep(1)
    assert e.value.status == P.PCA_ESTATE
    ctx.pca_reset(g, None)
    assert np.array_equal(ctx.state()[0], g)
    black = np.zeros((1, H, W), np.uint8)
    with pytest.raises(P.PcaError):
        ctx.pca_psnr_ssim(black, P.EST_LAST)
    # the estimate equal to the truth: MSE 0, PSNR +inf, SSIM 1
    p_eq, s_eq = ctx.pca_psnr_ssim(ctx.state(), P.EST_LAST)
    assert math.isinf(p_eq[0]) and p_eq[0] > 0 and abs(s_eq[0] - 1.0) < 1e-15
    # finalisation needs counted sweeps; a staged truth needs a non-NULL image
    with pytest.raises(P.PcaError, match="counted"):
        ctx.pca_finalize(g[None].copy())
    with pytest.raises(P.PcaError, match="NULL"):
        ctx.pca_stage_truth(None)
    # a row strip without NCCL: one PCA sweep per call, no Gibbs, no windowed SSIM
    strip = make_ctx(P.make_config(H, W, 2, row0=0, rows=8), g[:8])
    with pytest.raises(P.PcaError, match="one step"):
        strip.pca_sweep(2)
    with pytest.raises(P.PcaError, match="NCCL"):
        strip.pca_gibbs_sweep(1)
    # the context stays usable after argument errors (they do not poison it)
    ctx.pca_sweep(1)
    assert ctx.pca_get_stats().sweeps_done == 1


@pytest.mark.parametrize("kernel", [P.KERNEL_AUTO, P.KERNEL_GENERAL])
@pytest.mark.parametrize("levels", [2, 3, 5, 9, 16, 33])
@pytest.mark.parametrize("extreme", [dict(sigma=0.01), dict(q=1e6), dict(beta0=300.0),
                                     dict(sigma=0.02, q=500.0)])
def test_lockstep_extreme_parameters(cuda_device, kernel, levels, extreme):
    """Parameters whose factorised fp64 weights under/overflow (tiny sigma, huge q or beta):
    the binary tables and the general kernel's log-domain slow path still follow the oracle."""
    H, W = 24, 40
    g = synth.degrade(synth.smooth_labels(H, W, levels, 2), levels, 0.3, 3)
    cfg = P.make_config(H, W, levels, seed=17, kernel=kernel, **extreme)
    ctx = make_ctx(cfg, g, synth.random_labels((H, W), levels, 4))
    lockstep(ctx, cfg, 4).check(allow_rate=False)


def test_distribution_matches_exact_transition_powers(cuda_device):
    """50000 independent 3x3 torus chains (batch mode) after T sweeps from a fixed x0: the
    empirical state histogram matches delta_x0 P^T from exact enumeration (chi-square).
    Independent of the C oracle: pins the CUDA sampler to the paper's transition law."""
    from oracle import enumerate as en
    from test_oracle_pins import _chi2_ok

    B, T = 50000, 3
    lat = en.Lattice(3, 3, 2, nbhd=4, periodic=True)
    g = np.array([[0, 1, 0], [1, 1, 0], [0, 0, 1]], np.uint8)
    cfg = P.make_config(3, 3, 2, batch=B, neighborhood=4, periodic=True, sigma=0.5, beta0=1.25,
                        beta_step=0.0, seed=31337)
    ctx = make_ctx(cfg, np.broadcast_to(g, (B, 3, 3)).copy())
    ctx.pca_sweep(T)
    xs = ctx.state().reshape(B, 9).astype(np.int64)
    idx = (xs * (2 ** np.arange(8, -1, -1))).sum(1)
    hist = np.bincount(idx, minlength=512).astype(float)
    a, b, c = en.coefficients(1.25, 1 / 3, 0.51, 0.5)
    Pm = en.pca_matrix(lat, g.reshape(-1), a, b, c)
    row = np.zeros(512)
    row[en.state_index(lat, g.reshape(-1))] = 1.0
    for _ in range(T):
        row = row @ Pm
    ok, stat, crit = _chi2_ok(hist, row, B)
    assert ok, (stat, crit)


@pytest.mark.parametrize("H,W,nb,per", [(8192, 8192, 8, True), (4096, 32768, 8, True),
                                        (8192, 8192, 8, False), (8192, 8192, 4, True)],
                         ids=["c3", "c4-strip-shape", "c3-free", "c3-vn4"])
def test_full_size_sampled_rows(cuda_device, H, W, nb, per):
    """Bench-size lattices (config 3, 8192^2, and config 4's per-GPU 4096 x 32768 shape, l = 2,
    MPM on, one launch per sweep as in the bench): for EVERY one of four sweeps, rows sampled
    across the lattice (edges, middle, random) are recomputed by the oracle from the GPU's
    x_t; for config 3 the oracle recomputes the whole last sweep (67 M sites, ~5 s).  The MPM
    counts equal the sum of the four oracle-confirmed states at every site."""
    truth = synth.tiled_labels(H, W, 2, seed=1)
    g = synth.degrade(truth, 2, 0.5, seed=2)
    cfg = P.make_config(H, W, 2, neighborhood=nb, periodic=per, sigma=0.5, beta0=1.5,
                        beta_step=0.0, seed=11, mpm_burn_in=0)
    ctx = make_ctx(cfg, g)
    m = oracle_model(cfg)
    acc = np.zeros((H, W), np.uint16)
    tally = Tally()
    x = g
    rng = np.random.default_rng(0)
    for t in range(4):
        ctx.pca_sweep(1)
        xn = ctx.state()[0]
        rows = sorted({0, 1, H - 2, H - 1, H // 2} | set(rng.integers(0, H, 40).tolist()))
        for r in rows:
            ref, mg = orc.pca_sweep(m, x, g, 1.5, cfg.seed, 0, t, rows=(r, r + 1))
            tally.add(xn[r], ref[0], mg[0])
        acc += xn
        if t == 3 and H == W == 8192 and nb == 8 and per:
            ref, mg = orc.pca_sweep(m, x, g, 1.5, cfg.seed, 0, t)
            tally.add(xn, ref, mg)
        x = xn
    tally.check()
    assert np.array_equal(ctx.counts()[0], acc)


def test_config5_batch_full_size_sampled_chains(cuda_device):
    """Config 5 per GPU (128 chains of 512^2, l = 5, Moore-8, free, MPM on): whole chains
    sampled across the batch are recomputed by the oracle for the last sweep, and their
    planar counts equal the one-hot sums of the states."""
    B, H, W, L = 128, 512, 512, 5
    g = np.stack([synth.degrade(synth.smooth_labels(H, W, L, 7 + (b % 8)), L, 0.25, b) for b in range(B)])
    cfg = P.make_config(H, W, L, batch=B, sigma=0.25, seed=2025, mpm_burn_in=0)
    ctx = make_ctx(cfg, g)
    picks = [0, 1, 63, 100, 127]
    acc = np.zeros((len(picks), L, H, W), np.uint16)
    for _ in range(3):
        ctx.pca_sweep(1)
        xs = ctx.state()
        for i, b in enumerate(picks):
            acc[i] += (np.arange(L)[:, None, None] == xs[b][None]).astype(np.uint16)
    x3 = ctx.state()
    ctx.pca_sweep(1)
    x4 = ctx.state()
    m = oracle_model(cfg)
    tally = Tally()
    for i, b in enumerate(picks):
        ref, mg = orc.pca_sweep(m, x3[b], g[b], beta_of(cfg, 3), cfg.seed, b, 3)
        tally.add(x4[b], ref, mg)
        acc[i] += (np.arange(L)[:, None, None] == x4[b][None]).astype(np.uint16)
    tally.check()
    cnt = ctx.counts()
    for i, b in enumerate(picks):
        assert np.array_equal(cnt[b], acc[i])
    # fused finalisation over the whole batch vs the oracle's metrics on the picked chains
    truth = np.stack([synth.smooth_labels(H, W, L, 7 + (b % 8)) for b in range(B)])
    mpm = np.zeros((B, H, W), np.uint8)
    pf, sf = ctx.pca_finalize(truth, mpm)
    for i, b in enumerate(picks):
        cnt_o = acc[i].astype(np.uint32)
        assert np.array_equal(mpm[b], orc.mpm(cnt_o))
        for e, est in enumerate((x4[b], orc.mpm(cnt_o))):
            _, p_o, s_o, _ = orc.metrics(truth[b], est, L)
            assert abs(pf[b, e] - p_o) < 1e-9 and abs(sf[b, e] - s_o) < 1e-9


def test_nccl_loads_and_a_one_rank_communicator_attaches(cuda_device):
    """The NCCL plumbing of the strip path on the one GPU available: the unique id comes from
    the dlopen'ed libnccl, a one-rank communicator attaches (ncclCommInitRank) and a context
    with it sweeps and finalises like one without (one rank has no exchange and no
    all-reduce partner, so the chain must be unchanged)."""
    uid = P.pca_nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)
    H, W = 48, 80
    truth = synth.smooth_labels(H, W, 2, 3)
    g = synth.degrade(truth, 2, 0.5, 4)
    cfg = P.make_config(H, W, 2, periodic=True, sigma=0.5, seed=5, mpm_burn_in=0)
    a = make_ctx(cfg, g)
    a.pca_attach_nccl(uid, 1, 0)
    b = make_ctx(cfg, g)
    for ctx in (a, b):
        ctx.pca_sweep(7)
    assert np.array_equal(a.state(), b.state())
    assert np.array_equal(a.pca_finalize(truth[None])[0], b.pca_finalize(truth[None])[0])
    with pytest.raises(P.PcaError, match="already"):
        a.pca_attach_nccl(uid, 1, 0)
    a.pca_destroy()


@pytest.mark.parametrize("L", [2, 5])
def test_maximum_batch_of_tiny_lattices(cuda_device, L):
    """batch = 65535 (the grid-z limit) of 3x4 tori: sampled chains vs the oracle."""
    B, H, W = 65535, 3, 4
    g = np.random.default_rng(L).integers(0, L, (B, H, W)).astype(np.uint8)
    cfg = P.make_config(H, W, L, batch=B, neighborhood=8, periodic=True, sigma=0.4, seed=3,
                        mpm_burn_in=0)
    ctx = make_ctx(cfg, g)
    ctx.pca_sweep(2)
    x2 = ctx.state()
    ctx.pca_sweep(1)
    x3 = ctx.state()
    m = oracle_model(cfg)
    tally = Tally()
    for b in (0, 1, 777, 40000, B - 1):
        ref, mg = orc.pca_sweep(m, x2[b], g[b], beta_of(cfg, 2), cfg.seed, b, 2)
        tally.add(x3[b], ref, mg)
    tally.check(allow_rate=False)
    with pytest.raises(P.PcaError):
        P.PcaContext(P.make_config(H, W, L, batch=B + 1), np.zeros((B + 1, H, W), np.uint8))


@pytest.mark.parametrize("L,nb,per,ip", [(5, 8, False, 0), (3, 4, True, 2), (33, 8, False, 1),
                                         (2, 8, True, 0)])
def test_multi_sweep_launches_free_running_vs_oracle(cuda_device, L, nb, per, ip):
    """Small lattices run runs of sweeps in one cooperative launch (sweep_multi_kernel); the
    runs split at beta stages and at the burn-in.  Free-running against the oracle's chain:
    states and counts identical (no near-tie on these inputs)."""
    H, W = 24, 40
    truth = synth.smooth_labels(H, W, L, seed=L)
    g = synth.degrade(truth, L, 0.3, seed=L + 1)
    cfg = P.make_config(H, W, L, neighborhood=nb, periodic=per, sigma=0.3, beta0=1.0,
                        beta_step=0.25, beta_period=7, seed=41, mpm_burn_in=11, inertia_p=ip)
    ctx = make_ctx(cfg, g)
    ctx.pca_sweep(30)
    st = ctx.pca_get_stats()
    assert st.sweeps_done == 30 and st.counted_sweeps == 19
    assert st.sweep_launches < 30  # runs, not single sweeps
    x_o, cnt_o = orc.pca_run(oracle_model(cfg), g, g, 30, 1.0, 0.25, 7, 41, burn_in=11)
    assert np.array_equal(ctx.state()[0], x_o)
    c = ctx.counts()[0]
    assert np.array_equal(c, (cnt_o[1] if L == 2 else cnt_o).astype(np.uint16))


def _random_configs(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        L = int(rng.choice([2, 2, 3, 4, 5, 7, 9, 12, 16, 17, 33, 64, 100]))
        nb = int(rng.choice([4, 8]))
        per = bool(rng.integers(2))
        H = int(rng.integers(3 if per else 1, 70))
        W = int(rng.integers(3 if per else 1, 700))
        kw = dict(neighborhood=nb, periodic=per, sigma=float(rng.uniform(0.05, 0.8)),
                  q=float(rng.choice([0.0, 0.51, rng.uniform(0, 5)])), beta0=float(rng.uniform(0.3, 3)),
                  beta_step=float(rng.uniform(0, 1)), beta_period=int(rng.integers(1, 4)),
                  coef_scale=float(rng.choice([1.0, 0.5])), inertia_p=int(rng.integers(0, 3)),
                  J=float(rng.uniform(0.1, 1.0)), seed=int(rng.integers(1 << 40)),
                  chain0=int(rng.integers(0, 1000)), batch=int(rng.integers(1, 4)),
                  mpm_burn_in=int(rng.integers(-1, 3)),
                  kernel=int(rng.choice([P.KERNEL_AUTO, P.KERNEL_GENERAL])))
        out.append((H, W, L, kw))
    return out


@pytest.mark.parametrize("case", range(24))
def test_randomised_configurations_lockstep(cuda_device, case):
    """Random shapes, levels, neighbourhoods, boundaries, schedules, coefficients, inertia
    norms, batches and kernels: 4 lockstep sweeps against the oracle (R19 tolerance)."""
    H, W, L, kw = _random_configs(24, 2026)[case]
    cfg = P.make_config(H, W, L, **kw)
    B = kw["batch"]
    g = np.stack([synth.random_labels((H, W), L, seed=case * 10 + b) for b in range(B)])
    x0 = np.stack([synth.random_labels((H, W), L, seed=case * 10 + 5 + b) for b in range(B)])
    ctx = make_ctx(cfg, g, x0)
    lockstep(ctx, cfg, 4).check()


def test_restore_api_matches_the_step_by_step_calls(cuda_device):
    """paper_2507_14869_b200.api.restore (the paper protocol in one call) equals the explicit
    sequence of ABI calls and the oracle's chain."""
    from paper_2507_14869_b200.api import restore

    L, H, W = 5, 40, 56
    truth = synth.smooth_labels(H, W, L, seed=3)
    g = synth.degrade(truth, L, 0.25, seed=4)
    res = restore(g, L, truth=truth, sweeps=60, beta_period=20, seed=9, windowed=True)
    assert res.sweeps == 60 and res.counted_sweeps == 20
    cfg = P.make_config(H, W, L, sigma=0.25, beta_period=20, seed=9, mpm_burn_in=40)
    x_o, cnt_o = orc.pca_run(oracle_model(cfg), g, g, 60, 1.25, 0.25, 20, 9, burn_in=40)
    assert np.array_equal(res.last[0], x_o) and np.array_equal(res.mpm[0], orc.mpm(cnt_o))
    for e, est in enumerate((x_o, orc.mpm(cnt_o))):
        _, p_o, s_o, _ = orc.metrics(truth, est, L)
        assert abs(res.psnr[0, e] - p_o) < 1e-9 and abs(res.ssim[0, e] - s_o) < 1e-9
        assert abs(res.ssim_windowed[0, e] - orc.ssim_windowed(truth, est, L)) < 1e-12
    gb = restore(g, L, method="gibbs", sweeps=30, beta_period=20, seed=9)
    x_g, _ = orc.gibbs_run(oracle_model(cfg), g, g, 30, 1.25, 0.25, 20, 9, order="colour")
    assert np.array_equal(gb.last[0], x_g)


@pytest.mark.parametrize("shape,L,n", [((64, 64, 4, True), 2, 1), ((37, 531, 8, False), 2, 3),
                                       ((40, 130, 8, False), 5, 1), ((600, 600, 8, True), 5, 2)])
def test_changed_sites_counts_the_last_sweep(cuda_device, shape, L, n):
    """pca_changed_sites = number of sites with x_t != x_{t-1} (the double buffer), per chain,
    after single-sweep and multi-sweep launches; unavailable after a reset."""
    H, W, nb, per = shape
    B = 2
    g = np.stack([synth.random_labels((H, W), L, seed=b) for b in range(B)])
    cfg = P.make_config(H, W, L, batch=B, neighborhood=nb, periodic=per, sigma=0.4, seed=8)
    ctx = make_ctx(cfg, g)
    with pytest.raises(P.PcaError, match="previous"):
        ctx.pca_changed_sites()
    ctx.pca_sweep(4)
    prev = ctx.state()
    ctx.pca_sweep(n)
    if n > 1:
        m = oracle_model(cfg)
        x = prev
        for t in range(4, 4 + n - 1):
            x = np.stack([orc.pca_sweep(m, x[b], g[b], beta_of(cfg, t), cfg.seed, b, t)[0] for b in range(B)])
        prev = x
    cur = ctx.state()
    assert np.array_equal(ctx.pca_changed_sites(), (cur != prev).reshape(B, -1).sum(1))
    ctx.pca_reset(None, None)
    with pytest.raises(P.PcaError):
        ctx.pca_changed_sites()


@pytest.mark.parametrize("W", [64, 77, 200])
def test_packed_io_matches_dense_io(cuda_device, W):
    """packed_io (two levels): bit-packed g / x0 / truth in, bit-packed LAST / MPM / state out,
    host and device buffers, staged truth -- the same chain and metrics as dense I/O."""
    import torch

    H, B = 40, 2
    truth = np.stack([synth.smooth_labels(H, W, 2, seed=b) for b in range(B)])
    g = np.stack([synth.degrade(truth[b], 2, 0.5, seed=9 + b) for b in range(B)])
    kw = dict(batch=B, neighborhood=8, periodic=False, sigma=0.5, seed=17, mpm_burn_in=3)
    dense = make_ctx(P.make_config(H, W, 2, **kw), g)
    packed = P.PcaContext(P.make_config(H, W, 2, packed_io=1, **kw),
                          torch.from_numpy(P.pack_bits(g)).cuda())
    for c in (dense, packed):
        c.pca_sweep(9)
    assert np.array_equal(P.unpack_bits(packed.state(), W), dense.state())
    assert np.array_equal(P.unpack_bits(packed.estimate(P.EST_MPM), W), dense.estimate(P.EST_MPM))
    assert np.array_equal(packed.counts(), dense.counts())
    mpm_d = np.zeros((B, H, W), np.uint8)
    pd, sd = dense.pca_finalize(truth, mpm_d)
    mpm_p = torch.zeros((B, H, (W + 7) // 8), dtype=torch.uint8, device="cuda")
    pp, sp = packed.pca_finalize(torch.from_numpy(P.pack_bits(truth)).cuda(), mpm_p)
    assert np.array_equal(pp, pd) and np.array_equal(sp, sd)
    assert np.array_equal(P.unpack_bits(mpm_p.cpu().numpy(), W), mpm_d)
    packed.pca_stage_truth(P.pack_bits(truth))
    assert np.array_equal(packed.pca_finalize(None)[0], pd)
    # write a packed state and continue: same as the dense context written with the same state
    x = synth.random_labels((B, H, W), 2, seed=3)
    packed.pca_write_state(P.pack_bits(x))
    dense.pca_write_state(x)
    for c in (dense, packed):
        c.pca_sweep(2)
    assert np.array_equal(P.unpack_bits(packed.state(), W), dense.state())


@pytest.mark.parametrize("world", [2, 3])
def test_batch_mode_ranks_equal_one_context(cuda_device, world):
    """Batch mode (replicas only): splitting the chains over `world` rank
    contexts (dist.batch_context; here in one process, the contexts never wait on each other)
    gives every chain the same trajectory, counts and metrics as one context holding them
    all -- the chain0 offset keys the Philox words by global chain index."""
    from paper_2507_14869_b200 import dist as pdist

    n, H, W, L = 7, 40, 72, 5
    truth = np.stack([synth.smooth_labels(H, W, L, seed=10 + c % 3) for c in range(n)])
    g = np.stack([synth.degrade(truth[c], L, 0.25, seed=50 + c) for c in range(n)])
    kw = dict(sigma=0.25, beta_period=6, mpm_burn_in=8, seed=77)
    whole = P.PcaContext(P.make_config(H, W, L, batch=n, **kw), g)
    whole.pca_sweep(14)
    psnr_w, ssim_w = whole.pca_finalize(truth)
    x_w, c_w = whole.state(), whole.counts()
    psnr, ssim = np.zeros((n, 2)), np.zeros((n, 2))
    for r in range(world):
        ctx, c0 = pdist.batch_context(kw, H, W, L, g, n, world=world, rank=r)
        b = ctx.cfg.batch
        ctx.pca_sweep(14)
        psnr[c0:c0 + b], ssim[c0:c0 + b] = ctx.pca_finalize(truth[c0:c0 + b])
        assert np.array_equal(ctx.state(), x_w[c0:c0 + b])
        assert np.array_equal(ctx.counts(), c_w[c0:c0 + b])
        ctx.pca_destroy()
    assert np.array_equal(psnr, psnr_w) and np.array_equal(ssim, ssim_w)


def test_contexts_driven_from_concurrent_host_threads(cuda_device):
    """Independent contexts may be driven from several host threads at once (ctypes drops
    the GIL around every ABI call; the per-device launch caches initialise under a lock):
    each thread's chain equals the same chain run alone."""
    import threading

    shapes = [(48, 96, 2, 8, True), (40, 72, 5, 8, False), (34, 64, 9, 4, True), (64, 128, 2, 4, False)]
    def run(shape, out, i):
        H, W, L, nb, per = shape
        cfg = P.make_config(H, W, L, neighborhood=nb, periodic=per, sigma=0.3, seed=100 + i,
                            mpm_burn_in=3, beta_period=4)
        g = synth.degrade(synth.smooth_labels(H, W, L, seed=i), L, 0.3, seed=20 + i)
        ctx = P.PcaContext(cfg, g)
        ctx.pca_sweep(9)
        ctx.pca_gibbs_sweep(2)
        out[i] = (ctx.state(), ctx.counts())
        ctx.pca_destroy()

    alone = {}
    for i, sh in enumerate(shapes):
        run(sh, alone, i)
    together = {}
    threads = [threading.Thread(target=run, args=(sh, together, i)) for i, sh in enumerate(shapes)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for i in range(len(shapes)):
        assert np.array_equal(alone[i][0], together[i][0]) and np.array_equal(alone[i][1], together[i][1])


@pytest.mark.parametrize("packed", [0, 1])
def test_staged_input_reset_equals_direct_reset(cuda_device, packed):
    """pca_stage_input + pca_reset_staged (the copy on the copy stream, overlapping the sweeps
    enqueued after it) is pca_reset with that g: same chain, counts and metrics; host and
    device sources; an unstaged reset is an error."""
    import torch

    H, W = 40, 77
    g1 = synth.degrade(synth.smooth_labels(H, W, 2, 3), 2, 0.4, 4)[None]
    g2 = synth.degrade(synth.smooth_labels(H, W, 2, 5), 2, 0.4, 6)[None]
    enc = (lambda a: P.pack_bits(a)) if packed else (lambda a: a)
    kw = dict(sigma=0.4, seed=5, mpm_burn_in=2, packed_io=packed)
    a = P.PcaContext(P.make_config(H, W, 2, **kw), np.ascontiguousarray(enc(g1)))
    b = P.PcaContext(P.make_config(H, W, 2, **kw), np.ascontiguousarray(enc(g1)))
    with pytest.raises(P.PcaError, match="staged"):
        b.pca_reset_staged()
    for src in (np.ascontiguousarray(enc(g2)), torch.from_numpy(np.ascontiguousarray(enc(g1))).cuda()):
        b.pca_stage_input(src)
        b.pca_sweep(3)                # the copy overlaps these sweeps
        b.pca_reset_staged()
        a.pca_reset(src)
        a.pca_sweep(6)
        b.pca_sweep(6)
        assert np.array_equal(a.state(), b.state()) and np.array_equal(a.counts(), b.counts())


@pytest.mark.parametrize("packed", [0, 1])
def test_staged_temporary_pinned_input_survives_host_reuse(cuda_device, packed):
    """A temporary pinned tensor handed to pca_stage_input and dropped by the caller right
    away stays referenced by the binding until a host synchronisation covers its copy
    (ADVICE r1): new pinned tensors allocated and overwritten before pca_sync cannot reuse
    its block under the in-flight copy, so the chain starts from the staged g."""
    import torch

    H, W = 64, 400
    g1 = synth.degrade(synth.smooth_labels(H, W, 2, 3), 2, 0.4, 4)[None]
    g2 = synth.degrade(synth.smooth_labels(H, W, 2, 7), 2, 0.4, 8)[None]
    enc = (lambda a: P.pack_bits(a)) if packed else (lambda a: a)
    kw = dict(sigma=0.4, seed=5, mpm_burn_in=2, packed_io=packed)
    a = P.PcaContext(P.make_config(H, W, 2, **kw), np.ascontiguousarray(enc(g2)))
    b = P.PcaContext(P.make_config(H, W, 2, **kw), np.ascontiguousarray(enc(g1)))
    b.pca_sweep(20)
    tmp = torch.from_numpy(np.ascontiguousarray(enc(g2))).pin_memory()
    b.pca_stage_input(tmp)
    del tmp
    b.pca_reset_staged()
    junk = [torch.full(enc(g2).shape, 1 if packed else 0xAB, dtype=torch.uint8).pin_memory()
            for _ in range(8)]
    for j in junk:
        j.fill_(0xFF)
    b.pca_sweep(5)
    b.pca_sync()
    a.pca_sweep(5)
    assert np.array_equal(a.state(), b.state()) and np.array_equal(a.counts(), b.counts())


@pytest.mark.parametrize("packed", [0, 1])
def test_reset_with_new_g_equals_a_fresh_context(cuda_device, packed):
    """the fused reset (pca_reset(g_new, NULL) on a context that has swept) equals
    a fresh PcaContext(cfg, g_new): torus and free boundary, W in {64, 77}, 2 and 5 levels."""
    for periodic in (True, False):
        for W in (64, 77):
            for L in ((2,) if packed else (2, 5)):
                H = 40
                g1 = synth.degrade(synth.smooth_labels(H, W, L, 3), L, 0.3, 4)[None]
                g2 = synth.degrade(synth.smooth_labels(H, W, L, 5), L, 0.3, 6)[None]
                enc = (lambda a: P.pack_bits(a)) if packed else (lambda a: a)
                cfg = P.make_config(H, W, L, periodic=periodic, sigma=0.3, seed=9, mpm_burn_in=1,
                                    packed_io=packed)
                old = P.PcaContext(cfg, np.ascontiguousarray(enc(g1)))
                old.pca_sweep(7)
                old.pca_reset(np.ascontiguousarray(enc(g2)), None)
                new = P.PcaContext(cfg, np.ascontiguousarray(enc(g2)))
                for c in (old, new):
                    c.pca_sweep(6)
                assert np.array_equal(old.state(), new.state())
                assert np.array_equal(old.counts(), new.counts())
                truth = np.ascontiguousarray(enc(synth.smooth_labels(H, W, L, 5)[None]))
                assert np.array_equal(old.pca_finalize(truth), new.pca_finalize(truth))
                old.pca_destroy()
                new.pca_destroy()


@pytest.mark.parametrize("packed", [0, 1])
def test_finalize_async_equals_finalize(cuda_device, packed):
    """pca_finalize_async (the MPM image's device->host copy on the copy stream, overlapping
    the next run's reset and sweeps) gives pca_finalize's metrics and, after pca_sync, its
    image, run after run into the same pinned buffer; an estimate issued while a copy is in
    flight waits for it and is itself correct."""
    import torch

    H, W = 48, 83
    truth = synth.smooth_labels(H, W, 2, 7)[None]
    gs = [synth.degrade(truth[0], 2, 0.45, s)[None] for s in (8, 9, 10)]
    enc = (lambda a: P.pack_bits(a)) if packed else (lambda a: a)
    kw = dict(sigma=0.45, seed=11, mpm_burn_in=1, packed_io=packed)
    a = P.PcaContext(P.make_config(H, W, 2, **kw), np.ascontiguousarray(enc(gs[0])))
    b = P.PcaContext(P.make_config(H, W, 2, **kw), np.ascontiguousarray(enc(gs[0])))
    t_h = torch.from_numpy(np.ascontiguousarray(enc(truth))).pin_memory()
    out_a = np.zeros(t_h.shape, np.uint8)
    out_b = torch.zeros(tuple(t_h.shape), dtype=torch.uint8).pin_memory()
    for i, g in enumerate(gs):
        a.pca_reset(np.ascontiguousarray(enc(g)))
        a.pca_sweep(5 + i)
        pa, sa = a.pca_finalize(t_h.numpy(), out_a)
        if i:  # the previous run's image copy may still be in flight: reset/sweep overlap it
            b.pca_reset(np.ascontiguousarray(enc(g)))
        b.pca_sweep(5 + i)
        pb, sb = b.pca_finalize_async(t_h, out_b)
        assert np.array_equal(pa, pb) and np.array_equal(sa, sb)
        est = np.zeros(t_h.shape, np.uint8)
        b.pca_estimate(P.EST_MPM, est)  # reuses the output staging: waits for the copy
        b.pca_sync()
        assert np.array_equal(out_b.numpy(), out_a) and np.array_equal(est, out_a)


def test_finalize_async_device_output_none_and_destroy_in_flight(cuda_device):
    """pca_finalize_async with a device mpm_out (written as by pca_finalize), with no image
    (metrics only), with a batch of ragged chains into pageable host memory, and a context
    destroyed while its image copy may still be in flight."""
    import torch

    H, W, B = 33, 70, 3
    truth = np.stack([synth.smooth_labels(H, W, 5, seed=30 + b) for b in range(B)])
    g = np.stack([synth.degrade(truth[b], 5, 0.25, seed=40 + b) for b in range(B)])
    kw = dict(batch=B, neighborhood=8, periodic=False, sigma=0.25, seed=23, mpm_burn_in=2)
    a = make_ctx(P.make_config(H, W, 5, **kw), g)
    b = make_ctx(P.make_config(H, W, 5, **kw), g)
    for c in (a, b):
        c.pca_sweep(6)
    ref = np.zeros((B, H, W), np.uint8)
    pa, sa = a.pca_finalize(truth, ref)
    dev = torch.zeros((B, H, W), dtype=torch.uint8, device="cuda")
    pb, sb = b.pca_finalize_async(truth, dev)
    assert np.array_equal(pa, pb) and np.array_equal(sa, sb)
    assert np.array_equal(dev.cpu().numpy(), ref)
    pn, sn = b.pca_finalize_async(truth, None)
    assert np.array_equal(pn, pa) and np.array_equal(sn, sa)
    host = np.zeros((B, H, W), np.uint8)  # pageable
    b.pca_finalize_async(truth, host)
    b.pca_sync()
    assert np.array_equal(host, ref)
    pinned = torch.zeros((B, H, W), dtype=torch.uint8).pin_memory()
    b.pca_sweep(1)
    b.pca_finalize_async(truth, pinned)
    b.pca_destroy()  # waits for the copy stream before releasing the context
    a.pca_sweep(1)
    a.pca_finalize(truth, ref)
    assert np.array_equal(pinned.numpy(), ref)


def test_largest_single_lattice_32768_squared(cuda_device):
    """Config 4's whole 32768 x 32768 torus (1.07e9 sites, the P = 8 lattice) in ONE context on
    one GPU (~10 GB of workspace of the 180 GB): sampled rows of the last of four sweeps
    recomputed by the oracle from the GPU's x_t, and the MPM counts equal the sum of the four
    states at every site."""
    H = W = 32768
    g = synth.tiled_labels(H, W, 2, seed=21)  # a smooth two-level field as the observation
    cfg = P.make_config(H, W, 2, neighborhood=8, periodic=True, sigma=0.5, beta0=1.5,
                        beta_step=0.0, seed=13, mpm_burn_in=0)
    ctx = P.PcaContext(cfg, g[None])
    acc = np.zeros((H, W), np.uint16)
    for _ in range(3):
        ctx.pca_sweep(1)
        acc += ctx.state()[0]
    x3 = ctx.state()[0]
    ctx.pca_sweep(1)
    x4 = ctx.state()[0]
    acc += x4
    m = oracle_model(cfg)
    rows = sorted({0, 1, H - 1, H // 2} | set(np.random.default_rng(3).integers(0, H, 6).tolist()))
    tally = Tally()
    for r in rows:
        ref, mg = orc.pca_sweep(m, x3, g, 1.5, cfg.seed, 0, 3, rows=(r, r + 1))
        tally.add(x4[r], ref[0], mg[0])
    tally.check()
    assert np.array_equal(ctx.counts()[0], acc)
    ctx.pca_destroy()


def _random_new_kernel_configs(n, seed):
    """Random configurations for the round-2 kernels: PACKED (two levels, W a multiple of 512)
    and TABLE (3..5 levels), with extreme coefficients among them (the table kernel then
    hands those beta stages to the general kernel's log-domain path)."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        packed = i % 2 == 0
        L = 2 if packed else int(rng.choice([3, 4, 5]))
        nb = int(rng.choice([4, 8]))
        per = bool(rng.integers(2))
        H = int(rng.integers(3, 40))
        W = int(rng.choice([512, 1024, 1536])) if packed else int(rng.integers(3 if per else 1, 700))
        sigma = float(rng.choice([rng.uniform(0.05, 0.8), 0.01]))  # 0.01: b = 5000, weights underflow
        kw = dict(neighborhood=nb, periodic=per, sigma=sigma,
                  q=float(rng.choice([0.0, 0.51, rng.uniform(0, 5)])), beta0=float(rng.uniform(0.3, 3)),
                  beta_step=float(rng.uniform(0, 1)), beta_period=int(rng.integers(1, 4)),
                  coef_scale=float(rng.choice([1.0, 0.5])), inertia_p=int(rng.integers(0, 3)),
                  J=float(rng.uniform(0.1, 1.0)), seed=int(rng.integers(1 << 40)),
                  chain0=int(rng.integers(0, 1000)), batch=int(rng.integers(1, 4)),
                  mpm_burn_in=int(rng.integers(-1, 3)),
                  kernel=P.KERNEL_PACKED if packed else P.KERNEL_TABLE)
        out.append((H, W, L, kw))
    return out


@pytest.mark.parametrize("case", range(16))
def test_randomised_new_kernel_configurations_lockstep(cuda_device, case):
    """4 lockstep sweeps of the packed / table kernels against the oracle on random
    configurations (smooth states with random sprinkles: table rows and queued sites)."""
    H, W, L, kw = _random_new_kernel_configs(16, 77)[case]
    cfg = P.make_config(H, W, L, **kw)
    B = kw["batch"]
    g = np.stack([synth.random_labels((H, W), L, seed=case * 10 + b) for b in range(B)])
    x0 = np.stack([synth.smooth_labels(H, W, L, seed=case * 10 + 5 + b) for b in range(B)])
    x0[:, ::4, ::3] = synth.random_labels(x0[:, ::4, ::3].shape, L, seed=case)
    ctx = make_ctx(cfg, g, x0)
    assert ctx.pca_get_stats().kernel == kw["kernel"]
    lockstep(ctx, cfg, 4).check()
