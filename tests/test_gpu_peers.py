"""-m gpu: the device-initiated halo exchange (pca_attach_peers).

Strip contexts in ONE process share a stream here, so every phase a context waits for was
enqueued before the wait: nothing ever blocks on work that has not been issued, and no two
"ranks" wait on each other concurrently on the one GPU.  What this checks is the data path
(the sweep kernels' stores into the neighbours' halo rows, the pushes of a state load) and
the phase bookkeeping: the strips must reproduce the unsharded chain bit for bit.  The
cross-process mapping (CUDA IPC) is checked separately without any waiting."""
import numpy as np
import pytest

import oracle as orc
import paper_2507_14869_b200 as P
import synth
from parity_helpers import make_ctx, oracle_model

pytestmark = pytest.mark.gpu


def _strips(H, W, levels, bounds, base, g, stream):
    """Strip contexts for the row bounds; `stream`: one stream for all, or a list (one each)."""
    out = []
    for i in range(len(bounds) - 1):
        cfg = P.make_config(H, W, levels, row0=bounds[i], rows=bounds[i + 1] - bounds[i], **base)
        st = stream[i] if isinstance(stream, list) else stream
        out.append(P.PcaContext(cfg, np.ascontiguousarray(g[:, bounds[i]:bounds[i + 1]]), stream=st))
    return out


def _attach(strips, periodic):
    infos = [s.pca_peer_info() for s in strips]
    n = len(strips)
    for i, s in enumerate(strips):
        up = (i - 1) % n if periodic else i - 1
        dn = (i + 1) % n if periodic else i + 1
        s.pca_attach_peers(infos[up] if 0 <= up < n else None, infos[dn] if 0 <= dn < n else None)


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("levels,nb,batch", [(2, 8, 1), (2, 4, 2), (5, 8, 2), (33, 8, 1)])
def test_device_initiated_halos_reproduce_unsharded_chain(cuda_device, periodic, levels, nb, batch):
    import torch

    H, W = 48, 100
    g = np.stack([synth.degrade(synth.smooth_labels(H, W, levels, 5 + b), levels, 0.3, 6 + b)
                  for b in range(batch)])
    base = dict(neighborhood=nb, periodic=periodic, sigma=0.3, seed=99, mpm_burn_in=4, batch=batch,
                beta_period=5)
    full = P.PcaContext(P.make_config(H, W, levels, **base), g)
    stream = torch.cuda.Stream()
    bounds = [0, 17, 30, 48]
    strips = _strips(H, W, levels, bounds, base, g, stream)
    _attach(strips, periodic)
    launches0 = [s.pca_get_stats().sweep_launches for s in strips]
    for _ in range(12):
        for s in strips:
            s.pca_sweep(1)
    full.pca_sweep(12)
    for s, l0 in zip(strips, launches0):
        assert s.pca_get_stats().sweep_launches - l0 == 12  # one launch per sweep, no split
    got = np.concatenate([s.state() for s in strips], axis=1)
    assert np.array_equal(got, full.state())
    gc = np.concatenate([s.counts() for s in strips], axis=-2)
    assert np.array_equal(gc, full.counts())
    # and against the oracle's unsharded chains (chain id b per batch entry)
    for b in range(batch):
        x_o, cnt_o = orc.pca_run(oracle_model(full.cfg), g[b], g[b], 12, 1.25, 0.25, 5, 99, chain=b,
                                 burn_in=4)
        assert np.array_equal(got[b], x_o)
        assert np.array_equal(gc[b], (cnt_o[1] if levels == 2 else cnt_o).astype(np.uint16))
    # a state load (reset from a new x0) is a phase too: its edge rows are pushed
    x0 = np.stack([synth.random_labels((H, W), levels, 40 + b) for b in range(batch)])
    for i, s in enumerate(strips):
        s.pca_reset(None, np.ascontiguousarray(x0[:, bounds[i]:bounds[i + 1]]))
    full.pca_reset(None, x0)
    for _ in range(5):
        for s in strips:
            s.pca_sweep(1)
    full.pca_sweep(5)
    got = np.concatenate([s.state() for s in strips], axis=1)
    assert np.array_equal(got, full.state())
    for s in strips:
        s.pca_destroy()


def test_peer_attach_rejects_bad_uses(cuda_device):
    import torch

    H, W = 24, 40
    g = synth.random_labels((1, H, W), 2, 3)
    whole = P.PcaContext(P.make_config(H, W, 2), g)
    with pytest.raises(P.PcaError, match="row-strip"):
        whole.pca_attach_peers(whole.pca_peer_info(), None)
    stream = torch.cuda.Stream()
    a, b = _strips(H, W, 2, [0, 12, 24], dict(periodic=True, sigma=0.4), g, stream)
    with pytest.raises(P.PcaError, match="two peers"):
        a.pca_attach_peers(b.pca_peer_info(), None)
    other = P.PcaContext(P.make_config(H, W + 16, 2, row0=12, rows=12, periodic=True), synth.random_labels((1, 12, W + 16), 2, 1))
    with pytest.raises(P.PcaError, match="layout"):
        a.pca_attach_peers(other.pca_peer_info(), other.pca_peer_info())
    a.pca_attach_peers(b.pca_peer_info(), b.pca_peer_info())
    b.pca_attach_peers(a.pca_peer_info(), a.pca_peer_info())
    with pytest.raises(P.PcaError, match="already"):
        a.pca_attach_peers(b.pca_peer_info(), b.pca_peer_info())
    for c in (a, b, whole, other):
        c.pca_destroy()


def _ipc_owner(q_in, q_out, H, W):
    import torch

    torch.cuda.set_device(0)
    g = np.zeros((1, H, W), np.uint8)
    cfg = P.make_config(2 * H, W, 2, row0=0, rows=H)
    ctx = P.PcaContext(cfg, g)
    handle, off = ctx.pca_ipc_handle()
    q_out.put((handle, off))
    q_in.get(timeout=120)  # the other process has written our bottom halo rows
    h = ctx.pca_halo_ptrs()
    buf = torch.empty(h.row_bytes, dtype=torch.uint8, device="cuda")
    from test_gpu_parity import _cudart_memcpy
    _cudart_memcpy()(buf.data_ptr(), h.recv_bottom, h.row_bytes)
    q_out.put(buf.cpu().numpy().tobytes())
    ctx.pca_destroy()


def test_ipc_mapping_of_a_peer_workspace(cuda_device):
    """Process B maps process A's workspace through pca_ipc_handle / pca_open_peer and writes
    the two halo rows below A's strip through the mapped pointer; A reads exactly those bytes
    in its halo rows.  (No waiting between the processes.)"""
    import multiprocessing as mp

    import torch

    H, W = 16, 48
    ctx_mp = mp.get_context("spawn")
    q_in, q_out = ctx_mp.Queue(), ctx_mp.Queue()
    proc = ctx_mp.Process(target=_ipc_owner, args=(q_in, q_out, H, W))
    proc.start()
    try:
        handle, off = q_out.get(timeout=300)
        mine = P.PcaContext(P.make_config(2 * H, W, 2, row0=H, rows=H), np.zeros((1, H, W), np.uint8))
        peer_cfg = P.make_config(2 * H, W, 2, row0=0, rows=H)
        peer = mine.pca_open_peer(handle, off, peer_cfg)
        assert peer.rows == H and peer.batch == 1
        hb = mine.pca_halo_ptrs()
        pattern = (np.arange(hb.row_bytes) % 251).astype(np.uint8)
        src = torch.from_numpy(pattern).cuda()
        from test_gpu_parity import _cudart_memcpy
        pitch = hb.row_bytes // 2
        dst = peer.x[0] + (2 + H) * pitch  # rows H, H+1 of A's padded buffer 0 (below its strip)
        _cudart_memcpy()(dst, src.data_ptr(), hb.row_bytes)
        torch.cuda.synchronize()
        q_in.put(1)
        got = np.frombuffer(q_out.get(timeout=120), np.uint8)
        assert np.array_equal(got, pattern)
        P.pca_close_peer(peer)
        mine.pca_destroy()
    finally:
        proc.join(timeout=60)
        if proc.is_alive():
            proc.kill()


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("levels,nb,W", [(2, 8, 96), (2, 8, 90), (2, 4, 100), (5, 8, 96), (9, 4, 64)])
def test_gibbs_strips_over_peers_reproduce_unsharded_chain(cuda_device, periodic, levels, nb, W):
    """Row-strip Gibbs sweeps (binary TMA kernel, fused and 4-colour quad kernels) with the
    halo rows pushed to the peers after every launch reproduce the unsharded Gibbs chain, and
    PCA and Gibbs sweeps interleave on the same strips."""
    import torch

    H = 48
    if periodic and W % 2:
        pytest.skip("the Gibbs colouring needs an even torus")
    g = synth.degrade(synth.smooth_labels(H, W, levels, 8), levels, 0.3, 9)[None]
    base = dict(neighborhood=nb, periodic=periodic, sigma=0.3, seed=17, mpm_burn_in=3, beta_period=4)
    full = P.PcaContext(P.make_config(H, W, levels, **base), g)
    bounds = [0, 16, 31, 48]
    # one stream per strip, as on separate GPUs: a Gibbs sweep is several phases, and its
    # second phase waits for the neighbours' first, which they issue after this call returns
    # (on a shared stream that wait would sit in front of the work it waits for).  The waits
    # are stream waits, not spinning kernels, so the other strips' launches proceed.
    strips = _strips(H, W, levels, bounds, base, g, [torch.cuda.Stream() for _ in range(3)])
    _attach(strips, periodic)
    for step in range(8):
        for s in strips:
            (s.pca_gibbs_sweep if step % 3 else s.pca_sweep)(1)
    for step in range(8):
        (full.pca_gibbs_sweep if step % 3 else full.pca_sweep)(1)
    torch.cuda.synchronize()
    got = np.concatenate([s.state() for s in strips], axis=1)
    assert np.array_equal(got, full.state())
    gc = np.concatenate([s.counts() for s in strips], axis=-2)
    assert np.array_equal(gc, full.counts())
    # and against the oracle's sequence (colour-order Gibbs, R21, and PCA sweeps)
    m = oracle_model(full.cfg)
    x = g[0].copy()
    cnt = np.zeros((levels, H, W), np.int64)
    for t in range(8):
        beta = orc.beta_at(1.25, 0.25, 4, t)
        x = orc.gibbs_sweep_coloured(m, x, g[0], beta, 17, 0, t) if t % 3 else \
            orc.pca_sweep(m, x, g[0], beta, 17, 0, t)[0]
        if t >= 3:
            for k in range(levels):
                cnt[k] += x == k
    assert np.array_equal(got[0], x)
    assert np.array_equal(gc[0], (cnt[1] if levels == 2 else cnt).astype(np.uint16))
    for s in strips:
        s.pca_destroy()
