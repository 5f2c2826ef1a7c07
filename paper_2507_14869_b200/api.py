"""One-call restoration with the paper's protocol, built on the C ABI
binding: upload, n sweeps of the PCA (or of the checkerboard Gibbs sampler), the fused
finalisation (MPM image + PSNR/SSIM of the last sample and of MPM) and, on request, the
windowed SSIM.  Argument marshalling and call order only: every step runs in the library.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import (EST_LAST, EST_MPM, KERNEL_AUTO, PcaContext, make_config)


@dataclass
class Restoration:
    last: np.ndarray          # uint8 [batch][H][W]: the final sample
    mpm: np.ndarray           # uint8 [batch][H][W]: argmax of the counts (R15)
    psnr: np.ndarray | None   # [batch][2]: LAST, MPM (when truth is given)
    ssim: np.ndarray | None   # [batch][2]: global SSIM, LAST, MPM
    ssim_windowed: np.ndarray | None  # [batch][2]: 7x7 windowed SSIM, LAST, MPM
    sweeps: int
    counted_sweeps: int


def restore(noisy, levels: int, *, truth=None, method: str = "pca", sweeps: int = 1000,
            beta0: float = 1.25, beta_step: float = 0.25, beta_period: int = 250,
            burn_in: int | None = None, J: float = 1.0 / 3.0, q: float = 0.51,
            sigma: float = 0.25, neighborhood: int = 8, periodic: bool = False,
            coef_scale: float = 1.0, inertia_p: int = 0, seed: int = 0,
            kernel: int = KERNEL_AUTO, windowed: bool = False, device=None) -> Restoration:
    """Restore `noisy` (uint8 level indices, [H][W] or [batch][H][W]).

    Defaults are the paper's: J = 1/3, q = 0.51, Moore-8, free boundary, 1000 sweeps with
    beta = 1.25 + 0.25 every 250.  The MPM counts cover the last beta
    stage unless `burn_in` says otherwise.  method: "pca" (the synchronous lazy PCA) or
    "gibbs" (the checkerboard Gibbs sampler, R21).
    """
    if method not in ("pca", "gibbs"):
        raise ValueError("method must be 'pca' or 'gibbs'")
    g = np.ascontiguousarray(noisy, dtype=np.uint8)
    if g.ndim == 2:
        g = g[None]
    B, H, W = g.shape
    if burn_in is None:
        burn_in = max(0, sweeps - beta_period)
    if not 0 <= burn_in < sweeps:
        raise ValueError("need 0 <= burn_in < sweeps (the MPM estimate needs counted sweeps)")
    cfg = make_config(H, W, levels, batch=B, neighborhood=neighborhood, periodic=periodic, J=J,
                      q=q, sigma=sigma, beta0=beta0, beta_step=beta_step,
                      beta_period=beta_period, coef_scale=coef_scale, seed=seed,
                      mpm_burn_in=burn_in, kernel=kernel, inertia_p=inertia_p)
    ctx = PcaContext(cfg, g, device=device)
    try:
        tr = None
        if truth is not None:
            tr = np.ascontiguousarray(truth, dtype=np.uint8).reshape(B, H, W)
            ctx.pca_stage_truth(tr)  # uploads while the sweeps run
        (ctx.pca_sweep if method == "pca" else ctx.pca_gibbs_sweep)(sweeps)
        st = ctx.pca_get_stats()
        mpm = np.zeros((B, H, W), np.uint8)
        psnr = ssim = sw = None
        if tr is not None:
            psnr, ssim = ctx.pca_finalize(None, mpm)
            if windowed:
                sw = np.stack([ctx.pca_ssim_windowed(tr, EST_LAST),
                               ctx.pca_ssim_windowed(tr, EST_MPM)], axis=1)
        else:
            mpm = ctx.estimate(EST_MPM)
        last = ctx.state()
        return Restoration(last=last, mpm=mpm, psnr=psnr, ssim=ssim, ssim_windowed=sw,
                           sweeps=int(st.sweeps_done), counted_sweeps=int(st.counted_sweeps))
    finally:
        ctx.pca_destroy()
