"""Shared helpers for the -m gpu parity tests: run the CUDA path through the C ABI and
the oracle on the same seeded inputs, and classify every disagreement (R19)."""
from __future__ import annotations

import os

import numpy as np

import oracle as orc
import paper_2507_14869_b200 as P

MARGIN_TOL = 1e-6     # north star: exceptions only for draws within 1e-6 of a threshold
RATE_TOL = 1e-6       # ... and fewer than 1e-6 of all updates


def oracle_model(cfg: P.pca_config) -> orc.Model:
    return orc.model(cfg.height, cfg.width, cfg.levels, nbhd=cfg.neighborhood,
                     periodic=bool(cfg.periodic), J=cfg.J, q=cfg.q, sigma=cfg.sigma,
                     coef_scale=cfg.coef_scale, inertia_p=cfg.inertia_p)


def beta_of(cfg: P.pca_config, t: int) -> float:
    return orc.beta_at(cfg.beta0, cfg.beta_step, cfg.beta_period, t)


# every Tally of the session, written to gpurun_out/parity_report.json by conftest.py
REGISTRY: list = []


class Tally:
    def __init__(self, name: str = None):
        self.updates = 0
        self.mismatches = 0
        self.max_margin = 0.0
        self.name = name or os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
        self.counts = None  # lockstep(count_from=...): oracle-side MPM counts of the GPU states
        REGISTRY.append(self)

    def add(self, gpu_next, ora_next, margins):
        bad = gpu_next != ora_next
        self.updates += gpu_next.size
        n = int(bad.sum())
        if n:
            self.mismatches += n
            self.max_margin = max(self.max_margin, float(margins[bad].max()))
        return n

    def check(self, allow_rate=True):
        assert self.max_margin < MARGIN_TOL, (
            f"{self.mismatches} mismatches, one with oracle margin {self.max_margin:.3g} >= 1e-6")
        limit = RATE_TOL * self.updates if allow_rate else 0
        assert self.mismatches <= limit, (
            f"{self.mismatches} near-tie mismatches in {self.updates} updates (> 1e-6)")


def lockstep(ctx: P.PcaContext, cfg: P.pca_config, n: int, t0: int = 0, tally: Tally = None,
             count_from: int = None):
    """n sweeps in lockstep: at every sweep the oracle recomputes one sweep from the GPU's
    own x_t (state injection) and every site of the GPU's x_{t+1} is compared.
    count_from = the MPM burn-in: tally.counts[b][k] = #{t >= count_from: GPU x_{t+1} == k},
    the oracle's count rule (R15) applied to the lockstep states, so MPM and the metrics stay
    comparable when a near-tie mismatch makes the free-running chains part."""
    tally = tally or Tally()
    m = oracle_model(cfg)
    g = ctx._g_host
    x = ctx.state()
    if count_from is not None and tally.counts is None:
        tally.counts = np.zeros((cfg.batch, cfg.levels) + x.shape[1:], np.int64)
    for t in range(t0, t0 + n):
        ctx.pca_sweep(1)
        xn = ctx.state()
        for b in range(cfg.batch):
            ref, mg = orc.pca_sweep(m, x[b], g[b], beta_of(cfg, t), cfg.seed, cfg.chain0 + b, t)
            tally.add(xn[b], ref, mg)
            if count_from is not None and t >= count_from:
                for k in range(cfg.levels):
                    tally.counts[b, k] += xn[b] == k
        x = xn
    return tally


def make_ctx(cfg: P.pca_config, g: np.ndarray, x0: np.ndarray = None) -> P.PcaContext:
    g3 = g.reshape(cfg.batch, -1, cfg.width)
    ctx = P.PcaContext(cfg, np.ascontiguousarray(g3),
                       None if x0 is None else np.ascontiguousarray(x0.reshape(g3.shape)))
    ctx._g_host = g3
    return ctx
