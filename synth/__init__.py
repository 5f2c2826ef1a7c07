"""Seeded synthetic inputs shared by tests/ and bench.py.

This module holds none of the method's arithmetic (no PCA/Gibbs kernel, no metric): it
only makes label images shaped like the paper's workloads and degrades them with
Gaussian noise (section 6):

* ``smooth_labels``: Gaussian-smoothed white noise cut at quantiles into `levels`
  equal-area gray levels -- patchy images like the low-temperature MRF (Potts) samples of
  PAPER.md:496-500, without running a sampler;
* ``tiled_labels``: large images tiled from 512x512 smooth tiles with random flips
  (SURVEY.md 8(d) C3 recipe), cheap at 8192^2 and 32768^2;
* ``degrade``: add N(0, sigma^2) to each luminance k/(l-1), clamp to [0, 1], round to the
  nearest level with ties to the lower level (R12);
* ``random_labels``: i.i.d. uniform labels (random states for single-sweep parity).
"""
from __future__ import annotations

import numpy as np


def random_labels(shape, levels: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, levels, size=shape, dtype=np.uint8)


def smooth_labels(H: int, W: int, levels: int, seed: int, corr: float = 6.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal((H, W)).astype(np.float64)
    fy = np.fft.fftfreq(H)[:, None]
    fx = np.fft.rfftfreq(W)[None, :]
    kernel = np.exp(-2.0 * (np.pi * corr) ** 2 * (fx * fx + fy * fy))
    field = np.fft.irfft2(np.fft.rfft2(noise) * kernel, s=(H, W))
    qs = np.quantile(field, np.linspace(0, 1, levels + 1)[1:-1]) if levels > 1 else []
    return np.searchsorted(np.asarray(qs), field, side="right").astype(np.uint8)


def tiled_labels(H: int, W: int, levels: int, seed: int, tile: int = 512,
                 n_tiles: int = 4, corr: float = 6.0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    tiles = [smooth_labels(tile, tile, levels, seed * 1000 + k, corr) for k in range(n_tiles)]
    out = np.empty((H, W), np.uint8)
    for r in range(0, H, tile):
        for c in range(0, W, tile):
            t = tiles[rng.integers(n_tiles)]
            if rng.integers(2):
                t = t[::-1]
            if rng.integers(2):
                t = t[:, ::-1]
            out[r:r + tile, c:c + tile] = t[:min(tile, H - r), :min(tile, W - c)]
    return out


def degrade(truth: np.ndarray, levels: int, sigma: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    lum = truth.astype(np.float64) / (levels - 1)
    v = np.clip(lum + sigma * rng.standard_normal(truth.shape), 0.0, 1.0)
    f = v * (levels - 1)
    k = np.floor(f)
    k = k + ((f - k) > 0.5)
    return np.minimum(k, levels - 1).astype(np.uint8)
