"""Exact enumeration on tiny lattices (NumPy fp64) -- TEST INFRASTRUCTURE (see oracle/__init__).

Written independently of pca_oracle.c (no shared code).  Builds, for a lattice small
enough to list every configuration (l**n <= ~2**12 states):

* the PCA transition matrix P(x, w) = prod_i p_i(w_i; x)
  (eq. general_pca_definition) with the per-site law of PAPER.md:462-477 (R1);
* the Gibbs posterior pi_GS(a, b)(x) ∝ exp(a*Pairs(x) - D(x)), whose single-site
  conditionals are PAPER.md:417-429 (R4: the law the paper's Gibbs sampler samples);
* the PCA stationary law in closed form, pi~(x) ∝ exp(-D(x)) * prod_i Z_i(x)
  (eq. symm_ham_pca_stationary_measure, for the symmetric lifting
  H^(x,w) = -S(x,w) + D(x) + D(w), R2/R3), and as the literal double sum
  sum_w exp(-H^(x, w));
* the stationary vector of a matrix by a linear solve, TV distance, detailed-balance
  residual (eq. pca_detailed_balance), and the single-site Gibbs
  kernels K_i.

Sites are numbered i = r*W + c; a configuration is a length-n label vector and state
index = sum_i x_i * l**(n-1-i) (itertools.product order).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Lattice:
    H: int
    W: int
    levels: int
    nbhd: int = 8          # 8 = Moore; 4 = von Neumann
    periodic: bool = False  # False = free boundary

    @property
    def n(self) -> int:
        return self.H * self.W

    def neighbours(self) -> list[list[int]]:
        """F(r, c): Moore = max(|dr|, |dc|) = 1; von Neumann = |dr| + |dc| = 1."""
        if self.periodic:
            assert self.H >= 3 and self.W >= 3, "torus needs H, W >= 3 (distinct neighbours)"
        out = []
        for r in range(self.H):
            for c in range(self.W):
                lst = []
                for dr in (-1, 0, 1):
                    for dc in (-1, 0, 1):
                        cheb = max(abs(dr), abs(dc))
                        manh = abs(dr) + abs(dc)
                        ok = (cheb == 1) if self.nbhd == 8 else (manh == 1)
                        if not ok:
                            continue
                        rr, cc = r + dr, c + dc
                        if self.periodic:
                            rr %= self.H
                            cc %= self.W
                        elif not (0 <= rr < self.H and 0 <= cc < self.W):
                            continue
                        lst.append(rr * self.W + cc)
                out.append(lst)
        return out

    def states(self) -> np.ndarray:
        return np.array(list(itertools.product(range(self.levels), repeat=self.n)), dtype=np.int64)


def coefficients(beta, J, q, sigma, coef_scale=1.0):
    """a = 2*beta*J (prior), b = 1/(2 sigma^2) (data, not beta-scaled,
    PAPER.md:468 / R5), c = beta*q (inertia); coef_scale multiplies a, b."""
    return coef_scale * 2.0 * beta * J, coef_scale / (2.0 * sigma * sigma), beta * q


def luminance(levels):
    return np.arange(levels, dtype=np.float64) / (levels - 1)


def _dist2(lat: Lattice, g: np.ndarray) -> np.ndarray:
    """d2[i, s] = (lum g_i - lum s)^2."""
    L = luminance(lat.levels)
    return (L[np.asarray(g).reshape(-1)][:, None] - L[None, :]) ** 2


def inertia_penalty(lat: Lattice, p: int = 0) -> np.ndarray:
    """pen[x, s] = |lum x - lum s|^p with 0^0 = 0 (p = 0 is the paper's L0)."""
    L = luminance(lat.levels)
    d = np.abs(L[:, None] - L[None, :])
    pen = (d > 0).astype(float) if p == 0 else d ** p
    np.fill_diagonal(pen, 0.0)
    return pen


def _ncount(lat: Lattice, nbrs, x) -> np.ndarray:
    """cnt[i, s] = n_i(s; x)."""
    cnt = np.zeros((lat.n, lat.levels))
    for i in range(lat.n):
        for j in nbrs[i]:
            cnt[i, x[j]] += 1
    return cnt


def site_laws(lat: Lattice, x, g, a, b, c, inertia=True, p=0) -> np.ndarray:
    """p[i, s] for every site: softmax_s(a n_i(s;x) - b d_i(s)^2 - c |x_i - s|^p)."""
    nbrs = lat.neighbours()
    x = np.asarray(x).reshape(-1)
    E = a * _ncount(lat, nbrs, x) - b * _dist2(lat, g)
    if inertia:
        E = E - c * inertia_penalty(lat, p)[x]
    E = E - E.max(axis=1, keepdims=True)
    p = np.exp(E)
    return p / p.sum(axis=1, keepdims=True)


def pca_matrix(lat: Lattice, g, a, b, c, p=0) -> np.ndarray:
    """P[x, w] = prod_i p_i(w_i; x)."""
    S = lat.states()
    P = np.empty((len(S), len(S)))
    idx = np.arange(lat.n)
    for k, x in enumerate(S):
        laws = site_laws(lat, x, g, a, b, c, p=p)
        P[k] = np.prod(laws[idx[None, :], S], axis=1)
    return P


def pairs(lat: Lattice, x) -> int:
    """Number of agreeing unordered neighbour pairs {i, j}."""
    nbrs = lat.neighbours()
    x = np.asarray(x).reshape(-1)
    tot = 0
    for i in range(lat.n):
        for j in nbrs[i]:
            tot += int(x[i] == x[j])
    assert tot % 2 == 0
    return tot // 2


def data_term(lat: Lattice, x, g, b) -> float:
    """D(x) = b * sum_i (lum g_i - lum x_i)^2."""
    L = luminance(lat.levels)
    return float(b * np.sum((L[np.asarray(g).reshape(-1)] - L[np.asarray(x).reshape(-1)]) ** 2))


def gibbs_posterior(lat: Lattice, g, a, b) -> np.ndarray:
    """pi_GS(a, b)(x) ∝ exp(a Pairs(x) - D(x)); single-site conditionals = PAPER.md:417-429."""
    S = lat.states()
    logw = np.array([a * pairs(lat, x) - data_term(lat, x, g, b) for x in S])
    w = np.exp(logw - logw.max())
    return w / w.sum()


def pca_closed_form(lat: Lattice, g, a, b, c, p=0) -> np.ndarray:
    """pi~(x) ∝ exp(-D(x)) prod_i Z_i(x), Z_i(x) = sum_s exp(a n_i(s;x) - b d_i(s)^2 - c |x_i-s|^p)."""
    nbrs = lat.neighbours()
    S = lat.states()
    d2 = _dist2(lat, g)
    pen = inertia_penalty(lat, p)
    logw = np.empty(len(S))
    for k, x in enumerate(S):
        E = a * _ncount(lat, nbrs, x) - b * d2 - c * pen[x]
        logZ = np.log(np.exp(E).sum(axis=1)).sum()
        logw[k] = -data_term(lat, x, g, b) + logZ
    w = np.exp(logw - logw.max())
    return w / w.sum()


def pca_double_sum(lat: Lattice, g, a, b, c, p=0) -> np.ndarray:
    """pi(x) = sum_w exp(-H^(x,w)) / sum_{x,w} exp(-H^(x,w)) for
    H^(x, w) = -S(x, w) + D(x) + D(w),
    S(x, w) = a sum_i sum_{j in N(i)} 1{w_i = x_j} - c sum_i |w_i - x_i|^p."""
    nbrs = lat.neighbours()
    S = lat.states()
    pen = inertia_penalty(lat, p)
    D = np.array([data_term(lat, x, g, b) for x in S])
    Hm = np.empty((len(S), len(S)))
    for k, x in enumerate(S):
        s_xw = np.zeros(len(S))  # S(x, w) for every w (columns of S are w_i)
        for i in range(lat.n):
            for j in nbrs[i]:
                s_xw += a * (S[:, i] == x[j])
            s_xw -= c * pen[x[i], S[:, i]]
        Hm[k] = -s_xw + D[k] + D
    M = np.exp(-(Hm - Hm.min()))
    return M.sum(axis=1) / M.sum(), Hm


def stationary(P: np.ndarray) -> np.ndarray:
    """Left eigenvector pi P = pi, sum pi = 1, by a least-squares linear solve."""
    n = P.shape[0]
    A = np.vstack([P.T - np.eye(n), np.ones((1, n))])
    rhs = np.zeros(n + 1)
    rhs[-1] = 1.0
    pi, *_ = np.linalg.lstsq(A, rhs, rcond=None)
    return pi


def tv(p, q) -> float:
    return 0.5 * float(np.abs(np.asarray(p) - np.asarray(q)).sum())


def detailed_balance_residual(pi, P) -> float:
    F = pi[:, None] * P
    return float(np.abs(F - F.T).max())


def gibbs_site_kernel(lat: Lattice, g, a, b, i) -> np.ndarray:
    """K_i[x, x'] = pi(X_i = x'_i | rest of x) if x' differs from x only at site i."""
    S = lat.states()
    index = {tuple(s): k for k, s in enumerate(S)}
    K = np.zeros((len(S), len(S)))
    for k, x in enumerate(S):
        p = site_laws(lat, x, g, a, b, 0.0, inertia=False)[i]
        for s in range(lat.levels):
            y = x.copy()
            y[i] = s
            K[k, index[tuple(y)]] += p[s]
    return K


def state_index(lat: Lattice, x) -> int:
    k = 0
    for v in np.asarray(x).reshape(-1):
        k = k * lat.levels + int(v)
    return k
