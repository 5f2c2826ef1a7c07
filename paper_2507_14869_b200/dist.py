"""Host-side logic of the row-strip decomposition and of batch sharding.

* ``strip_rows``: balanced contiguous partition of the H global rows over the ranks.
* ``ring_peers``: the ranks above/below a strip (a ring on the torus; -1 at free ends).
* ``broadcast_unique_id``: rank 0 creates the NCCL unique id through the C ABI
  (pca_nccl_unique_id) and torch.distributed broadcasts its 128 bytes.
* ``strip_context``: a PcaContext for this rank's strip with NCCL attached.
* ``attach_peers_ipc``: the device-initiated halo exchange instead of NCCL sends/receives:
  every rank publishes its workspace's CUDA IPC handle, maps its up / down neighbours' and
  attaches them (pca_attach_peers).
* ``chain_range``: the batch-mode partition of independent chains (replicas only).
* ``batch_context``: a PcaContext for this rank's chain range (chain0 = its first global
  chain, so every chain draws the same Philox words whatever the world size).
* ``gather_chain_metrics``: the per-chain PSNR/SSIM of every rank, assembled on rank 0 in
  global chain order (C5's final gather).

The per-sweep halo exchange itself runs inside the library (runtime.cu ``exchange``):
after each sweep a rank sends its first owned row to ``up`` and its last to ``down`` and
receives the two halo rows -- the same protocol ``tests/test_dist_cpu.py`` replays with gloo.
"""
from __future__ import annotations


def strip_rows(H: int, world: int, rank: int) -> tuple[int, int]:
    """(row0, rows) of `rank`: the first H % world ranks get one extra row."""
    if world < 1 or not 0 <= rank < world or H < world:
        raise ValueError("need 0 <= rank < world <= H")
    base, extra = divmod(H, world)
    rows = base + (1 if rank < extra else 0)
    row0 = rank * base + min(rank, extra)
    return row0, rows


def ring_peers(rank: int, world: int, periodic: bool) -> tuple[int, int]:
    """(up, down): the ranks owning the rows just above / below this strip, -1 if none."""
    if periodic:
        return (rank - 1) % world, (rank + 1) % world
    return (rank - 1 if rank > 0 else -1), (rank + 1 if rank < world - 1 else -1)


def chain_range(n_chains: int, world: int, rank: int) -> tuple[int, int]:
    """(chain0, batch) of `rank` in batch mode: contiguous, balanced."""
    return strip_rows(n_chains, world, rank)


def broadcast_unique_id(group=None) -> bytes:
    import torch.distributed as dist

    from . import pca_nccl_unique_id

    obj = [pca_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    assert isinstance(obj[0], bytes) and len(obj[0]) == 128
    return obj[0]


def attach_peers_ipc(ctx, cfg_kwargs: dict, H: int, W: int, levels: int, group=None):
    """Map the up / down ranks' workspaces (CUDA IPC, exchanged with torch.distributed) and
    attach them to this rank's strip context: from then on every PCA sweep stores its edge rows
    straight into the neighbours' halo rows.  Returns the mapped peers (pca_close_peer them
    after the context is destroyed)."""
    import torch.distributed as dist

    from . import make_config

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    handle, off = ctx.pca_ipc_handle()
    table = [None] * world
    dist.all_gather_object(table, (handle, off), group=group)
    up, down = ring_peers(rank, world, bool(cfg_kwargs.get("periodic", False)))
    peers = {}
    for q in {up, down} - {-1}:
        row0, rows = strip_rows(H, world, q)
        cfg = make_config(H, W, levels, row0=row0, rows=rows, **cfg_kwargs)
        peers[q] = ctx.pca_open_peer(table[q][0], table[q][1], cfg)
    dist.barrier(group=group)  # every rank has mapped its neighbours before anyone pushes
    ctx.pca_attach_peers(peers.get(up), peers.get(down))
    return list(peers.values())


def strip_context(cfg_kwargs: dict, H: int, W: int, levels: int, g_strip, *, stream=None,
                  group=None):
    """Create this rank's strip context (rows from strip_rows) and attach NCCL."""
    import torch.distributed as dist

    from . import PcaContext, make_config

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    row0, rows = strip_rows(H, world, rank)
    cfg = make_config(H, W, levels, row0=row0, rows=rows if world > 1 else 0, **cfg_kwargs)
    ctx = PcaContext(cfg, g_strip, stream=stream)
    if world > 1:
        ctx.pca_attach_nccl(broadcast_unique_id(group), world, rank)
    return ctx


def batch_context(cfg_kwargs: dict, H: int, W: int, levels: int, g_all, n_chains: int, *,
                  world: int | None = None, rank: int | None = None, stream=None, group=None):
    """Batch mode (replicas only): this rank's contiguous range of the `n_chains` independent
    chains.  `g_all` holds every chain's observed image ([n_chains][H][W], host or device);
    only this rank's slice is uploaded.  Returns (context, chain0).  `world` / `rank` default
    to the process group's."""
    from . import PcaContext, make_config

    if world is None or rank is None:
        import torch.distributed as dist

        world, rank = dist.get_world_size(group), dist.get_rank(group)
    chain0, batch = chain_range(n_chains, world, rank)
    cfg = make_config(H, W, levels, batch=batch, chain0=chain0, **cfg_kwargs)
    return PcaContext(cfg, g_all[chain0:chain0 + batch], stream=stream), chain0


def gather_chain_metrics(chain0: int, psnr, ssim, n_chains: int, group=None):
    """Every rank passes its chain0 and its [batch][2] PSNR / SSIM arrays (LAST, MPM); rank 0
    returns the [n_chains][2] arrays in global chain order, the other ranks (None, None)."""
    import numpy as np
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    parts = [None] * world
    dist.all_gather_object(parts, (int(chain0), np.asarray(psnr), np.asarray(ssim)), group=group)
    if rank != 0:
        return None, None
    P = np.full((n_chains, 2), np.nan)
    S = np.full((n_chains, 2), np.nan)
    for c0, p, s in parts:
        P[c0:c0 + len(p)] = p
        S[c0:c0 + len(s)] = s
    if np.isnan(S).any():
        raise ValueError("the ranks' chain ranges do not cover every chain")
    return P, S
