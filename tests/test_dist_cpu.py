"""Multi-process (gloo, world size 2, CPU) coverage of the N > 1 host logic.

The row-strip protocol of paper_2507_14869_b200.dist (partition, ring peers, the NCCL
unique-id broadcast) is replayed with the CPU oracle as the per-strip sweep and gloo
send/recv as the halo transport: the gathered sharded chain must equal the unsharded
oracle chain bit for bit (the RNG is keyed by global row/col).
Rows a rank does not own are filled with random labels, so reading anything but the
exchanged halo rows would break the equality.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_2507_14869_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, H, W, levels, periodic, nsweeps, out_q, method="pca"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = pdist.broadcast_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert all(i == ids[0] for i in ids)

        row0, rows = pdist.strip_rows(H, world, rank)
        up, down = pdist.ring_peers(rank, world, periodic)
        rng = np.random.default_rng(100 + rank)
        g = np.random.default_rng(7).integers(0, levels, (H, W), dtype=np.uint8)
        m = orc.model(H, W, levels, nbhd=8, periodic=periodic, sigma=0.4)
        x = rng.integers(0, levels, (H, W), dtype=np.uint8)  # poison: rows not owned
        x[row0:row0 + rows] = g[row0:row0 + rows]            # x0 = g on the strip

        def exchange(x, depth=1):
            # library order: send(top -> up), recv(bottom halo <- down),
            #                send(bottom -> down), recv(top halo <- up); `depth` rows each
            reqs = []
            top = torch.from_numpy(x[row0:row0 + depth].copy())
            bot = torch.from_numpy(x[row0 + rows - depth:row0 + rows].copy())
            halo_bot = torch.empty((depth, W), dtype=torch.uint8)
            halo_top = torch.empty((depth, W), dtype=torch.uint8)
            if up >= 0:
                reqs.append(dist.isend(top, up, tag=0))
            if down >= 0:
                reqs.append(dist.irecv(halo_bot, down, tag=0))
                reqs.append(dist.isend(bot, down, tag=1))
            if up >= 0:
                reqs.append(dist.irecv(halo_top, up, tag=1))
            for r in reqs:
                r.wait()
            for d in range(depth):
                if up >= 0:
                    x[(row0 - depth + d) % H] = halo_top.numpy()[d]
                if down >= 0:
                    x[(row0 + rows + d) % H] = halo_bot.numpy()[d]

        if method == "pca2":
            # two sweeps per pass (sweeps_per_pass == 2): g is known on the strip only, its halo
            # rows come from the neighbours once; x halos are 2 rows deep, once per pass
            g_full = g
            g = np.random.default_rng(500 + rank).integers(0, levels, (H, W), dtype=np.uint8)
            g[row0:row0 + rows] = g_full[row0:row0 + rows]
            exchange(g)
            exchange(x, 2)
        else:
            exchange(x)
        for t in range(0, nsweeps, 2) if method == "pca2" else []:
            # sweep t on the strip and one row beyond each edge (from the 2-deep halo and the
            # g halo row), then sweep t+1 on the strip; one exchange per pass
            raw = [row0 - 1] + list(range(row0, row0 + rows)) + [row0 + rows]
            rows_t = [r % H for r in raw] if periodic else [r for r in raw if 0 <= r < H]
            y = rng.integers(0, levels, (H, W), dtype=np.uint8)
            for r in rows_t:
                y[r] = orc.pca_sweep(m, x, g, 1.25, 99, 0, t, rows=(r, r + 1))[0][0]
            new, _ = orc.pca_sweep(m, y, g, 1.25, 99, 0, t + 1, rows=(row0, row0 + rows))
            x = rng.integers(0, levels, (H, W), dtype=np.uint8)
            x[row0:row0 + rows] = new
            exchange(x, 2)
        for t in range(nsweeps) if method != "pca2" else []:
            if method == "pca":
                new, _ = orc.pca_sweep(m, x, g, 1.25, 99, 0, t, rows=(row0, row0 + rows))
                x = rng.integers(0, levels, (H, W), dtype=np.uint8)  # fresh poison every sweep
                x[row0:row0 + rows] = new
                exchange(x)
            else:  # Gibbs (runtime order, Moore-8 fused): the two colours of a row parity on
                # the strip (no exchange in between: they only meet within a row), then a halo
                # exchange; twice per sweep
                for par in range(2):
                    new = x
                    for k in (2 * par, 2 * par + 1):
                        new = orc.gibbs_colour_phase(m, new, g, 1.25, 99, 0, t, k, rows=(row0, row0 + rows))
                    x = rng.integers(0, levels, (H, W), dtype=np.uint8)
                    x[row0:row0 + rows] = new[row0:row0 + rows]
                    exchange(x)
        strips = [None] * world
        dist.all_gather_object(strips, (row0, x[row0:row0 + rows].copy()))
        if rank == 0:
            full = np.zeros((H, W), np.uint8)
            for r0, s in strips:
                full[r0:r0 + len(s)] = s
            g = np.random.default_rng(7).integers(0, levels, (H, W), dtype=np.uint8)
            ref = g.copy()
            for t in range(nsweeps):
                if method in ("pca", "pca2"):
                    ref, _ = orc.pca_sweep(m, ref, g, 1.25, 99, 0, t)
                else:
                    ref = orc.gibbs_sweep_coloured(m, ref, g, 1.25, 99, 0, t)
            out_q.put(bool(np.array_equal(full, ref)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("periodic", [True, False])
def test_two_rank_strip_exchange_reproduces_unsharded_chain(periodic):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 13, 11, 3, periodic, 6, q))
             for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok


@pytest.mark.parametrize("periodic", [True, False])
def test_two_rank_strips_two_sweeps_per_pass(periodic):
    """The temporally blocked strip protocol (sweeps_per_pass == 2): g halo
    rows exchanged once, x halos 2 rows deep exchanged once per pass, each pass recomputing
    sweep t one row beyond the strip: the unsharded chain, with half the exchanges."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 13, 11, 3, periodic, 6, q, "pca2"))
             for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok


@pytest.mark.parametrize("periodic", [True, False])
def test_two_rank_strip_gibbs_reproduces_unsharded_chain(periodic):
    """pca_gibbs_sweep's strip protocol (Moore-8): the two colours of each row parity on the
    owned rows, then a halo exchange, reproduces the unsharded colour-order scan (even torus
    sides)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    H, W = (14, 12) if periodic else (13, 11)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, H, W, 3, periodic, 5, q, "gibbs"))
             for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok


def test_partition_and_peers():
    for H in (3, 10, 4096 * 8, 17):
        for world in (1, 2, 3, 8):
            if world > H:
                continue
            spans = [pdist.strip_rows(H, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (a0, an), (b0, _) in zip(spans, spans[1:]):
                assert a0 + an == b0
            assert sum(n for _, n in spans) == H
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
    assert pdist.ring_peers(0, 4, True) == (3, 1)
    assert pdist.ring_peers(0, 4, False) == (-1, 1)
    assert pdist.ring_peers(3, 4, False) == (2, -1)
    assert pdist.ring_peers(0, 2, True) == (1, 1)
    assert pdist.chain_range(1024, 8, 3) == (384, 128)
    with pytest.raises(ValueError):
        pdist.strip_rows(2, 3, 0)


def _gather_worker(rank, world, port, n_chains, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        chain0, batch = pdist.chain_range(n_chains, world, rank)
        chains = np.arange(chain0, chain0 + batch, dtype=float)
        psnr = np.stack([chains, chains + 0.5], axis=1)       # a value that names its chain
        ssim = np.stack([chains / 100, chains / 100 + 0.005], axis=1)
        P, S = pdist.gather_chain_metrics(chain0, psnr, ssim, n_chains)
        if rank == 0:
            want = np.arange(n_chains, dtype=float)
            out_q.put(bool(np.array_equal(P[:, 0], want) and np.array_equal(P[:, 1], want + 0.5)
                           and np.allclose(S[:, 0], want / 100)))
        else:
            out_q.put(P is None and S is None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_chains", [(2, 7), (3, 1024)])
def test_batch_mode_gathers_chain_metrics_in_global_order(world, n_chains):
    """C5's final gather: each rank's chain range, metrics assembled on rank 0."""
    if world > n_chains:
        pytest.skip("fewer chains than ranks")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n_chains, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(res)


class _FakeStripCtx:
    """Stands in for a PcaContext in the host logic of dist.attach_peers_ipc."""

    def __init__(self, rank):
        self.rank = rank
        self.opened = []
        self.attached = None

    def pca_ipc_handle(self):
        return bytes([self.rank]) * 64, 1000 + self.rank

    def pca_open_peer(self, handle, off, cfg):
        self.opened.append((handle[0], off, cfg.row0, cfg.rows, cfg.height))
        return ("peer", handle[0])

    def pca_attach_peers(self, up, down):
        self.attached = (up, down)


def _peers_worker(rank, world, port, H, periodic, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = _FakeStripCtx(rank)
        pdist.attach_peers_ipc(ctx, dict(periodic=periodic, sigma=0.5), H, 64, 2)
        up, dn = pdist.ring_peers(rank, world, periodic)
        ok = ctx.attached == (("peer", up) if up >= 0 else None, ("peer", dn) if dn >= 0 else None)
        for h, off, row0, rows, height in ctx.opened:  # each neighbour's own strip and handle
            ok &= (row0, rows) == pdist.strip_rows(H, world, h) and off == 1000 + h and height == H
        ok &= sorted(h for h, *_ in ctx.opened) == sorted({up, dn} - {-1})
        out_q.put(bool(ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic", [(2, True), (3, True), (3, False)])
def test_attach_peers_ipc_maps_the_neighbour_strips(world, periodic):
    """dist.attach_peers_ipc: every rank publishes its workspace handle, maps exactly its up /
    down neighbours with THEIR strip configs, and attaches them in (up, down) order."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peers_worker, args=(r, world, port, 50, periodic, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(res)
