"""CPU oracle for arXiv 2507.14869 (lazy PCA posterior sampling) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2507_14869_b200`` never imports it and shares no code with it.

Two independent parts:

* ``pca_oracle.c`` (loaded here through ctypes): the plain single-threaded fp64
  implementation of the PCA sweep, the systematic Gibbs sampler, MPM counts,
  PSNR/SSIM, degradation and MRF synthesis.  Each C function cites its passage.
* ``enumerate.py``: exact enumeration of transition matrices and stationary laws on
  tiny lattices (NumPy, fp64), written separately from the C code.

The C library is compiled with gcc on first use (``build()``), without fast-math
and with FMA contraction off so that its fp64 arithmetic is the plain IEEE
evaluation of the formulas as written.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pca_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

TAG_PCA, TAG_GIBBS, TAG_NOISE, TAG_GEN_INIT, TAG_GEN_GIBBS = 1, 2, 3, 4, 5


def build(force: bool = False) -> str:
    """Compile pca_oracle.c into liboracle.so (gcc, -O2, IEEE fp64, no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
            "-fno-fast-math", "-Wall", "-o", tmp, _SRC, "-lm",
        ])
        os.replace(tmp, _LIB)
    return _LIB


class Model(ctypes.Structure):
    """Mirror of ``orc_model`` (pca_oracle.c)."""

    _fields_ = [
        ("H", ctypes.c_int), ("W", ctypes.c_int), ("levels", ctypes.c_int),
        ("nbhd", ctypes.c_int), ("periodic", ctypes.c_int),
        ("J", ctypes.c_double), ("q", ctypes.c_double), ("sigma", ctypes.c_double),
        ("coef_scale", ctypes.c_double), ("inertia_p", ctypes.c_int),
    ]


def model(H, W, levels, nbhd=8, periodic=False, J=1.0 / 3.0, q=0.51, sigma=0.25,
          coef_scale=1.0, inertia_p=0) -> Model:
    return Model(int(H), int(W), int(levels), int(nbhd), int(bool(periodic)), float(J),
                 float(q), float(sigma), float(coef_scale), int(inertia_p))


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER
        u8p, u32p, f64p = P(ctypes.c_uint8), P(ctypes.c_uint32), P(ctypes.c_double)
        mp = P(Model)
        sig = {
            "orc_philox4x32_10": (None, [u32p, u32p, u32p]),
            "orc_draw": (ctypes.c_uint32, [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]),
            "orc_beta_at": (ctypes.c_double, [ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                              ctypes.c_int]),
            "orc_pca_site_probs": (None, [mp, u8p, u8p, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, f64p]),
            "orc_gibbs_site_probs": (None, [mp, u8p, u8p, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_double, f64p]),
            "orc_decide": (ctypes.c_int, [f64p, ctypes.c_int, ctypes.c_double, f64p]),
            "orc_pca_sweep_rows": (None, [mp, u8p, u8p, u8p, f64p, ctypes.c_double,
                                          ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                          ctypes.c_int, ctypes.c_int]),
            "orc_pca_sweep": (None, [mp, u8p, u8p, u8p, f64p, ctypes.c_double, ctypes.c_uint64,
                                     ctypes.c_uint32, ctypes.c_uint32]),
            "orc_pca_run": (None, [mp, u8p, u8p, u32p, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                   ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int]),
            "orc_gibbs_sweep": (None, [mp, u8p, u8p, ctypes.c_double, ctypes.c_uint64,
                                       ctypes.c_uint32, ctypes.c_uint32]),
            "orc_gibbs_run": (None, [mp, u8p, u8p, u32p, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                     ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                                     ctypes.c_int]),
            "orc_gibbs_sweep_coloured": (None, [mp, u8p, u8p, ctypes.c_double, ctypes.c_uint64,
                                                ctypes.c_uint32, ctypes.c_uint32]),
            "orc_gibbs_colour": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
            "orc_gibbs_colour_phase": (None, [mp, u8p, u8p, ctypes.c_double, ctypes.c_uint64,
                                              ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int]),
            "orc_mpm": (None, [u32p, ctypes.c_int, ctypes.c_size_t, u8p]),
            "orc_metrics": (ctypes.c_int, [u8p, u8p, ctypes.c_size_t, ctypes.c_int, f64p, f64p,
                                           f64p]),
            "orc_ssim_windowed": (ctypes.c_double, [u8p, u8p, ctypes.c_int, ctypes.c_int,
                                                    ctypes.c_int]),
            "orc_quantize": (ctypes.c_int, [ctypes.c_double, ctypes.c_int]),
            "orc_gauss": (ctypes.c_double, [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                            ctypes.c_uint32]),
            "orc_degrade": (None, [u8p, u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_uint64, ctypes.c_uint32]),
            "orc_generate_mrf": (None, [mp, u8p, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_uint64, ctypes.c_uint32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray, ct):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a


# ---------------------------------------------------------------------------
def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c, ctypes.c_uint32), _p(k, ctypes.c_uint32),
                            _p(out, ctypes.c_uint32))
    return out


def draw(seed, tag, chain, t, row, col) -> int:
    return int(lib().orc_draw(seed, tag, chain, t, row, col))


def beta_at(beta0, beta_step, period, t) -> float:
    return float(lib().orc_beta_at(beta0, beta_step, period, t))


def pca_site_probs(m: Model, x, g, r, c, beta):
    x, g = _u8(x), _u8(g)
    p = np.zeros(m.levels, np.float64)
    lib().orc_pca_site_probs(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8),
                             r, c, beta, _p(p, ctypes.c_double))
    return p


def gibbs_site_probs(m: Model, x, g, r, c, beta):
    x, g = _u8(x), _u8(g)
    p = np.zeros(m.levels, np.float64)
    lib().orc_gibbs_site_probs(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8),
                               r, c, beta, _p(p, ctypes.c_double))
    return p


def decide(p, u):
    p = np.ascontiguousarray(p, np.float64)
    mg = ctypes.c_double(0.0)
    w = lib().orc_decide(_p(p, ctypes.c_double), len(p), float(u), ctypes.byref(mg))
    return int(w), float(mg.value)


def pca_sweep(m: Model, x, g, beta, seed, chain, t, rows=None):
    """One sweep; returns (new_state, margins).  rows=(r0, r1) restricts the update to
    those rows and returns only them: (new_rows [r1-r0, W], margins [r1-r0, W])."""
    x, g = _u8(x), _u8(g)
    if rows is None:
        out = x.copy()
        mg = np.full(x.shape, np.inf, np.float64)
        lib().orc_pca_sweep_rows(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8),
                                 _p(out, ctypes.c_uint8), _p(mg, ctypes.c_double), beta, seed,
                                 chain, t, 0, m.H)
        return out, mg
    r0, r1 = rows
    out = np.zeros((r1 - r0, m.W), np.uint8)
    mg = np.full((r1 - r0, m.W), np.inf, np.float64)
    # the C routine writes out[r*W + c] for r in [r0, r1): hand it base pointers shifted back
    # by r0 rows so that only the small buffers are touched
    outp = ctypes.cast(out.ctypes.data - r0 * m.W, ctypes.POINTER(ctypes.c_uint8))
    mgp = ctypes.cast(mg.ctypes.data - r0 * m.W * 8, ctypes.POINTER(ctypes.c_double))
    lib().orc_pca_sweep_rows(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8), outp,
                             mgp, beta, seed, chain, t, r0, r1)
    return out, mg


def pca_run(m: Model, x0, g, n, beta0, beta_step, period, seed, chain=0, t0=0, burn_in=-1):
    """n PCA sweeps from x0 (sweep indices t0..t0+n-1).  Returns (x_n, counts[l][H][W])."""
    x = _u8(x0).copy()
    g = _u8(g)
    counts = np.zeros((m.levels,) + x.shape, np.uint32)
    lib().orc_pca_run(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8),
                      _p(counts, ctypes.c_uint32), t0, n, beta0, beta_step, period, seed, chain,
                      burn_in)
    return x, counts


def gibbs_sweep(m: Model, x, g, beta, seed, chain, t):
    x = _u8(x).copy()
    g = _u8(g)
    lib().orc_gibbs_sweep(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8), beta,
                          seed, chain, t)
    return x


def gibbs_sweep_coloured(m: Model, x, g, beta, seed, chain, t):
    """One Gibbs sweep in checkerboard colour order (see orc_gibbs_colour)."""
    x = _u8(x).copy()
    g = _u8(g)
    lib().orc_gibbs_sweep_coloured(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8),
                                   beta, seed, chain, t)
    return x


def gibbs_colour_phase(m: Model, x, g, beta, seed, chain, t, k, rows=None):
    """Colour k of the colour-order scan over rows [r0, r1) (default all), in place on a copy."""
    x = _u8(x).copy()
    g = _u8(g)
    r0, r1 = rows if rows is not None else (0, m.H)
    lib().orc_gibbs_colour_phase(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8),
                                 beta, seed, chain, t, k, r0, r1)
    return x


def gibbs_colour(nbhd, r, c) -> int:
    return int(lib().orc_gibbs_colour(nbhd, r, c))


def gibbs_run(m: Model, x0, g, n, beta0, beta_step, period, seed, chain=0, t0=0, burn_in=-1,
              order="column"):
    """order: "column" = the paper's column-major scan, "colour" = the
    checkerboard colour order of the GPU Gibbs sampler."""
    x = _u8(x0).copy()
    g = _u8(g)
    counts = np.zeros((m.levels,) + x.shape, np.uint32)
    lib().orc_gibbs_run(ctypes.byref(m), _p(x, ctypes.c_uint8), _p(g, ctypes.c_uint8),
                        _p(counts, ctypes.c_uint32), t0, n, beta0, beta_step, period, seed, chain,
                        burn_in, {"column": 0, "colour": 1}[order])
    return x, counts


def mpm(counts):
    counts = np.ascontiguousarray(counts, np.uint32)
    levels = counts.shape[0]
    N = counts[0].size
    out = np.zeros(counts.shape[1:], np.uint8)
    lib().orc_mpm(_p(counts, ctypes.c_uint32), levels, N, _p(out, ctypes.c_uint8))
    return out


def metrics(truth, y, levels):
    """(mse, psnr, ssim_global, status) of restored y against the original truth."""
    truth, y = _u8(truth), _u8(y)
    mse, psnr, ssim = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    st = lib().orc_metrics(_p(truth, ctypes.c_uint8), _p(y, ctypes.c_uint8), truth.size, levels,
                           ctypes.byref(mse), ctypes.byref(psnr), ctypes.byref(ssim))
    return mse.value, psnr.value, ssim.value, st


def ssim_windowed(truth, y, levels):
    truth, y = _u8(truth), _u8(y)
    H, W = truth.shape
    return float(lib().orc_ssim_windowed(_p(truth, ctypes.c_uint8), _p(y, ctypes.c_uint8), H, W,
                                         levels))


def quantize(v, levels) -> int:
    return int(lib().orc_quantize(float(v), levels))


def gauss(seed, chain, row, col) -> float:
    return float(lib().orc_gauss(seed, chain, row, col))


def degrade(x, levels, sigma, seed, chain=0):
    x = _u8(x)
    H, W = x.shape
    out = np.zeros_like(x)
    lib().orc_degrade(_p(x, ctypes.c_uint8), _p(out, ctypes.c_uint8), H, W, levels, sigma, seed,
                      chain)
    return out


def generate_mrf(m: Model, n, beta_start, beta_end, seed, chain=0):
    x = np.zeros((m.H, m.W), np.uint8)
    lib().orc_generate_mrf(ctypes.byref(m), _p(x, ctypes.c_uint8), n, beta_start, beta_end, seed,
                           chain)
    return x
