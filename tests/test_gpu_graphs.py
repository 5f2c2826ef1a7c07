"""-m gpu: CUDA-graph-captured sweep runs (pca_config.graphs): a pca_sweep(n) run is captured
once per starting host state and replayed when it recurs; the chain, counts and metrics must
be those of the same calls without graphs, and recurring runs must be replays."""
import numpy as np
import pytest

import oracle as orc
import paper_2507_14869_b200 as P
import synth
from parity_helpers import oracle_model

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kernel,W,spp", [(P.KERNEL_PACKED, 1024, 0), (P.KERNEL_BINARY, 1040, 0),
                                          (P.KERNEL_BINARY, 1040, 2), (P.KERNEL_GENERAL, 1040, 0)])
def test_graph_replayed_runs_equal_direct_runs(cuda_device, kernel, W, spp):
    H = 300
    truth = synth.smooth_labels(H, W, 2, seed=4)
    g = synth.degrade(truth, 2, 0.45, seed=5)
    kw = dict(periodic=True, sigma=0.45, beta0=1.1, beta_step=0.3, beta_period=9, seed=6, mpm_burn_in=7,
              kernel=kernel, sweeps_per_pass=spp)
    a = P.PcaContext(P.make_config(H, W, 2, graphs=1, **kw), g[None].copy())
    b = P.PcaContext(P.make_config(H, W, 2, **kw), g[None].copy())
    results = []
    for step in range(3):          # the bench's step: reset, a run of sweeps, finalisation
        for c in (a, b):
            c.pca_reset(None, None)
            c.pca_sweep(20)        # crosses two beta stages and the burn-in
            c.pca_sweep(5)
        assert np.array_equal(a.state(), b.state()) and np.array_equal(a.counts(), b.counts())
        pa = a.pca_finalize(truth[None], np.zeros((1, H, W), np.uint8))
        pb = b.pca_finalize(truth[None], np.zeros((1, H, W), np.uint8))
        assert np.array_equal(pa[0], pb[0]) and np.array_equal(pa[1], pb[1])
        results.append(a.state()[0])
    st = a.pca_get_stats()
    # steps 2 and 3 replay both runs; the packed kernel's first run of step 1 also packed g (a
    # different starting state: g not yet packed), so its step-2 run is one more capture
    assert st.graph_replays == (3 if kernel == P.KERNEL_PACKED else 4)
    assert st.sweeps_done == 25 and st.counted_sweeps == 18
    x_o, cnt_o = orc.pca_run(oracle_model(a.cfg), g, g, 25, 1.1, 0.3, 9, 6, burn_in=7)
    assert np.array_equal(results[-1], x_o) and np.array_equal(a.counts()[0], cnt_o[1].astype(np.uint16))
    # a new g invalidates nothing it should not: the packed kernel repacks g inside the run
    g2 = np.ascontiguousarray(g[::-1])
    for c in (a, b):
        c.pca_reset(g2[None].copy(), None)
        c.pca_sweep(20)
    assert np.array_equal(a.state(), b.state()) and np.array_equal(a.counts(), b.counts())


def test_graphs_rejected_for_more_levels(cuda_device):
    with pytest.raises(P.PcaError):
        P.pca_workspace_bytes(P.make_config(64, 64, 5, graphs=1))


def test_graph_captured_strip_sweeps_with_loopback_halos(cuda_device):
    """Row-strip contexts with graphs: each pca_sweep(1) of a strip is captured (the strip
    path's launches; the caller exchanges the halos between calls) and the strips reproduce
    the oracle's unsharded chain.  (With NCCL attached the captured run also holds the halo
    sends / receives; with peers attached graphs are not used.)"""
    import torch

    from test_gpu_parity import _cudart_memcpy

    copy = _cudart_memcpy()
    H, W, Pn = 48, 1040, 3
    g = synth.degrade(synth.smooth_labels(H, W, 2, 5), 2, 0.4, 6)
    base = dict(neighborhood=8, periodic=True, sigma=0.4, seed=3, mpm_burn_in=2, graphs=1)
    b = [0, 17, 30, 48]
    strips = [P.PcaContext(P.make_config(H, W, 2, row0=b[i], rows=b[i + 1] - b[i], **base),
                           np.ascontiguousarray(g[b[i]:b[i + 1]])[None]) for i in range(Pn)]

    def exchange():
        torch.cuda.synchronize()
        hs = [s.pca_halo_ptrs() for s in strips]
        for i in range(Pn):
            up, dn = (i - 1) % Pn, (i + 1) % Pn
            copy(hs[i].recv_top, hs[up].send_bottom, hs[i].row_bytes)
            copy(hs[i].recv_bottom, hs[dn].send_top, hs[i].row_bytes)
        torch.cuda.synchronize()

    exchange()
    for _ in range(8):
        for s in strips:
            s.pca_sweep(1)
        exchange()
    got = np.concatenate([s.state()[0] for s in strips], axis=0)
    x_o, cnt_o = orc.pca_run(oracle_model(P.make_config(H, W, 2, **base)), g, g, 8, 1.25, 0.25, 250, 3,
                             burn_in=2)
    assert np.array_equal(got, x_o)
    assert np.array_equal(np.concatenate([s.counts()[0] for s in strips], axis=0), cnt_o[1].astype(np.uint16))
