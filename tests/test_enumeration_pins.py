"""Pins for oracle/enumerate.py against what the paper and the mathematics fix.

Every check compares the enumeration with something other than itself: the paper's
stationary-law theorem, detailed balance, exact special cases
(bipartite q = 0 factorisation, complete-graph mean-field law, one-site closed form,
label-flip symmetry), Gibbs invariance and the q -> infinity limit
(read through R4 in DESIGN.md).
"""
from math import comb

import numpy as np
import pytest

from oracle import enumerate as en

RNG = np.random.default_rng(20250714)

INSTANCES = [
    # (lattice, g, beta, sigma)
    (en.Lattice(3, 3, 2, nbhd=4, periodic=True), np.array([0, 1, 0, 1, 0, 1, 0, 1, 0]), 1.25, 0.5),
    (en.Lattice(3, 3, 2, nbhd=8, periodic=False), RNG.integers(0, 2, 9), 1.0, 0.5),
    (en.Lattice(2, 2, 3, nbhd=8, periodic=False), np.array([0, 2, 1, 2]), 1.25, 0.4),
    (en.Lattice(1, 3, 4, nbhd=8, periodic=False), np.array([3, 0, 2]), 1.5, 0.3),
]


@pytest.mark.parametrize("lat,g,beta,sigma", INSTANCES)
@pytest.mark.parametrize("q", [0.0, 0.51, 2.0])
def test_stationary_law_closed_form(lat, g, beta, sigma, q):
    """for a symmetric pair Hamiltonian the chain is reversible with
    stationary law Z_x/Z.  The transition matrix built site-by-site must (i) be row
    stochastic, (ii) have that closed form as its stationary vector, (iii) satisfy
    detailed balance, and (iv) agree with the literal double sum over w."""
    a, b, c = en.coefficients(beta, 1 / 3, q, sigma)
    P = en.pca_matrix(lat, g, a, b, c)
    assert np.abs(P.sum(axis=1) - 1).max() < 1e-13
    assert P.min() > 0  # irreducible + aperiodic
    cf = en.pca_closed_form(lat, g, a, b, c)
    pi = en.stationary(P)
    assert en.tv(pi, cf) < 1e-10
    assert en.detailed_balance_residual(cf, P) < 1e-15
    ds, Hm = en.pca_double_sum(lat, g, a, b, c)
    assert np.abs(Hm - Hm.T).max() < 1e-12  # the lifting H^ is symmetric
    assert en.tv(ds, cf) < 1e-12


def test_q_limit_is_gibbs_with_doubled_coefficients():
    """PAPER.md:320-322 ("improves as q grows"), read via R4: the q -> inf limit of the
    literal PCA is pi_GS(2a, 2b); TV decreases monotonically to ~0.  It does NOT tend to
    pi_GS(a, b) (the law of the paper's own Gibbs sampler)."""
    lat, g, beta, sigma = INSTANCES[0]
    tv2, tv1 = [], []
    for q in [0, 0.51, 1, 2, 4, 8, 16]:
        a, b, c = en.coefficients(beta, 1 / 3, q, sigma)
        cf = en.pca_closed_form(lat, g, a, b, c)
        tv2.append(en.tv(cf, en.gibbs_posterior(lat, g, 2 * a, 2 * b)))
        tv1.append(en.tv(cf, en.gibbs_posterior(lat, g, a, b)))
    assert all(x > y for x, y in zip(tv2, tv2[1:]))
    assert tv2[-1] < 1e-7
    assert tv1[-1] > 0.3


def test_matched_mode_limit_is_paper_gibbs():
    """coef_scale = 0.5 halves a and b (R4 'matched' mode): the limit is pi_GS(a, b)."""
    lat, g, beta, sigma = INSTANCES[0]
    tvs = []
    for q in [0.51, 2, 4, 8, 16]:
        ah, bh, c = en.coefficients(beta, 1 / 3, q, sigma, coef_scale=0.5)
        cf = en.pca_closed_form(lat, g, ah, bh, c)
        tvs.append(en.tv(cf, en.gibbs_posterior(lat, g, 2 * ah, 2 * bh)))
    assert all(x > y for x, y in zip(tvs, tvs[1:]))
    assert tvs[-1] < 1e-7


@pytest.mark.parametrize("lat", [en.Lattice(3, 3, 2, nbhd=4), en.Lattice(2, 3, 3, nbhd=4)])
def test_bipartite_q0_factorises_into_checkerboard_gibbs(lat):
    """q = 0 on a bipartite graph (4-neighbour, free): new even sites depend only on old
    odd sites and vice versa, so the PCA is two interleaved exact checkerboard Gibbs
    samplers and pi~ = (even marginal of pi_GS) x (odd marginal of pi_GS)."""
    g = RNG.integers(0, lat.levels, lat.n)
    a, b, c = en.coefficients(1.25, 1 / 3, 0.0, 0.5)
    cf = en.pca_closed_form(lat, g, a, b, c)
    gs = en.gibbs_posterior(lat, g, a, b)
    S = lat.states()
    even = np.array([(i // lat.W + i % lat.W) % 2 == 0 for i in range(lat.n)])
    key_e = [tuple(s[even]) for s in S]
    key_o = [tuple(s[~even]) for s in S]
    me, mo = {}, {}
    for k in range(len(S)):
        me[key_e[k]] = me.get(key_e[k], 0.0) + gs[k]
        mo[key_o[k]] = mo.get(key_o[k], 0.0) + gs[k]
    prod = np.array([me[key_e[k]] * mo[key_o[k]] for k in range(len(S))])
    assert en.tv(cf, prod) < 1e-13
    P = en.pca_matrix(lat, g, a, b, c)
    assert en.tv(en.stationary(P), prod) < 1e-10


def test_complete_graph_mean_field():
    """3x3 Moore torus = complete graph K9: at zero field pi_GS ∝ exp(a sum_k C(m_k, 2)),
    m_k = number of sites with label k (pins the pair counting)."""
    lat = en.Lattice(3, 3, 2, nbhd=8, periodic=True)
    g = np.zeros(9, int)
    a = 0.7
    gs = en.gibbs_posterior(lat, g, a, 0.0)
    S = lat.states()
    logw = np.array([a * sum(comb(int((s == k).sum()), 2) for k in range(2)) for s in S])
    ref = np.exp(logw - logw.max())
    ref /= ref.sum()
    assert en.tv(gs, ref) < 1e-14


def test_label_flip_symmetry():
    """Zero field (b = 0): P(x, w) = P(1-x, 1-w) exactly.  With a field the symmetry
    holds under the joint reflection (x, g) -> (l-1-x, l-1-g)."""
    lat = en.Lattice(3, 3, 2, nbhd=4, periodic=True)
    S = lat.states()
    flip = np.array([en.state_index(lat, 1 - s) for s in S])
    g = RNG.integers(0, 2, 9)
    a, _, c = en.coefficients(1.25, 1 / 3, 0.51, 0.5)
    P0 = en.pca_matrix(lat, g, a, 0.0, c)
    assert np.abs(P0 - P0[np.ix_(flip, flip)]).max() < 1e-15
    a, b, c = en.coefficients(1.25, 1 / 3, 0.51, 0.5)
    lat3 = en.Lattice(2, 2, 3, nbhd=8)
    g3 = np.array([0, 1, 2, 2])
    S3 = lat3.states()
    refl = np.array([en.state_index(lat3, 2 - s) for s in S3])
    P = en.pca_matrix(lat3, g3, a, b, c)
    Pr = en.pca_matrix(lat3, 2 - g3, a, b, c)
    assert np.abs(P - Pr[np.ix_(refl, refl)]).max() < 1e-15
    assert np.abs(P - P[np.ix_(refl, refl)]).max() > 1e-3  # the field does break plain flip


@pytest.mark.parametrize("q", [0.0, 0.51, 3.0])
def test_one_site_closed_form(q):
    """1x1 lattice (no neighbours): pi~(x) ∝ e^{-d(x)} (e^{-d(x)} + e^{-c} sum_{s!=x} e^{-d(s)});
    at c = 0 it is the single-site posterior e^{-d(x)}/sum."""
    lat = en.Lattice(1, 1, 4)
    g = np.array([1])
    a, b, c = en.coefficients(1.5, 1 / 3, q, 0.4)
    d = b * (np.array([1 / 3]) - np.arange(4) / 3) ** 2
    ref = np.array([np.exp(-d[x]) * (np.exp(-d[x]) + np.exp(-c) * (np.exp(-d).sum() - np.exp(-d[x])))
                    for x in range(4)])
    ref /= ref.sum()
    P = en.pca_matrix(lat, g, a, b, c)
    assert en.tv(en.stationary(P), ref) < 1e-12
    if q == 0.0:
        post = np.exp(-d) / np.exp(-d).sum()
        assert en.tv(ref, post) < 1e-15


@pytest.mark.parametrize("lat,g,beta,sigma", INSTANCES[:3])
def test_gibbs_single_site_kernels_leave_posterior_invariant(lat, g, beta, sigma):
    """each single-site Gibbs update (conditional of PAPER.md:417-429)
    leaves pi_GS(a, b) invariant, hence so does the systematic sweep."""
    a, b, _ = en.coefficients(beta, 1 / 3, 0.0, sigma)
    gs = en.gibbs_posterior(lat, g, a, b)
    for i in range(lat.n):
        K = en.gibbs_site_kernel(lat, g, a, b, i)
        assert np.abs(K.sum(axis=1) - 1).max() < 1e-13
        assert np.abs(gs @ K - gs).max() < 1e-15


def test_large_q_freezes():
    """Infinite inertia freezes the chain: P -> I (SPEC.md:436 style)."""
    lat, g, beta, sigma = INSTANCES[0]
    a, b, c = en.coefficients(1.0, 1 / 3, 50.0, sigma)
    P = en.pca_matrix(lat, g, a, b, c)
    assert np.abs(P - np.eye(len(P))).max() < 1e-6


def test_tv_arithmetic():
    assert en.tv([0.5, 0.5], [0.9, 0.1]) == pytest.approx(0.4, abs=1e-15)
    assert en.tv([1, 0], [0, 1]) == 1.0


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("lat,g", [(en.Lattice(2, 2, 3, nbhd=8), np.array([0, 2, 1, 2])),
                                   (en.Lattice(1, 3, 4, nbhd=8), np.array([3, 0, 2])),
                                   (en.Lattice(2, 3, 3, nbhd=4), np.array([2, 0, 1, 1, 2, 0]))])
def test_l1_l2_inertia_keep_the_closed_form(lat, g, p):
    """PAPER.md:279 / 483-485: the inertia q sum_i |x_i - w_i|^p (p = 1, 2) is symmetric in
    (x, w), so the stationary law is still exp(-D) prod_i Z_i."""
    a, b, c = en.coefficients(1.25, 1 / 3, 0.9, 0.4)
    P = en.pca_matrix(lat, g, a, b, c, p=p)
    cf = en.pca_closed_form(lat, g, a, b, c, p=p)
    assert en.tv(en.stationary(P), cf) < 1e-10
    assert en.detailed_balance_residual(cf, P) < 1e-15
    ds, Hm = en.pca_double_sum(lat, g, a, b, c, p=p)
    assert np.abs(Hm - Hm.T).max() < 1e-12 and en.tv(ds, cf) < 1e-12
    P0 = en.pca_matrix(lat, g, a, b, c, p=0)
    assert np.abs(P - P0).max() > 1e-3  # the norm matters for l > 2


def test_inertia_norm_irrelevant_for_two_levels():
    """For l = 2 every change costs |1 - 0|^p = 1: L0, L1 and L2 inertia coincide."""
    lat = en.Lattice(3, 3, 2, nbhd=8)
    g = RNG.integers(0, 2, 9)
    a, b, c = en.coefficients(1.25, 1 / 3, 0.51, 0.5)
    P0 = en.pca_matrix(lat, g, a, b, c, p=0)
    for p in (1, 2):
        assert np.abs(en.pca_matrix(lat, g, a, b, c, p=p) - P0).max() == 0.0
