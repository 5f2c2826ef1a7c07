"""Pins for the C oracle (oracle/pca_oracle.c) against what the paper and mathematics fix.

- Philox: Random123 known-answer vectors (tests/golden/philox4x32_10_kat.txt).
- Annealing schedule and score arithmetic: PAPER.md:508 and PAPER.md:466-468
  (tests/golden/paper_worked_values.txt).
- Per-site laws vs the independently written exact-enumeration module (which is itself
  pinned to the paper's stationary-law theorem in test_enumeration_pins.py).
- Sampling: one-step frequencies of the C sweep vs the exact transition matrix;
  long-run histograms of the C PCA chain vs the closed-form stationary law pi~ and of
  the C Gibbs chain vs pi_GS.
- Metrics: PAPER.md:516-534 special cases; degradation: Gaussian-CDF closed forms.
"""
import math
import os

import numpy as np
import pytest

import oracle as orc
from oracle import enumerate as en

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_values():
    vals = {}
    for line in open(os.path.join(GOLD, "paper_worked_values.txt")):
        line = line.split("#")[0].strip()
        if line:
            k, v = line.split("=")
            vals[k.strip()] = float(v)
    return vals


GV = _golden_values()


def test_philox_known_answers():
    rows = [l.split() for l in open(os.path.join(GOLD, "philox4x32_10_kat.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(h, 16) for h in r]
        out = orc.philox4x32_10(v[0:4], v[4:6])
        assert [int(o) for o in out] == v[6:10]


def test_draw_counter_layout():
    """RNG contract: key = (seed lo, seed hi); ctr = (col>>2, row, t, tag<<24 | chain);
    word col & 3."""
    seed = 0x0123456789ABCDEF
    for (tag, chain, t, row, col) in [(1, 0, 0, 0, 0), (1, 7, 3, 11, 13), (2, 0xFFFFFF, 999, 8191, 8190)]:
        out = orc.philox4x32_10([col >> 2, row, t, (tag << 24) | chain],
                                [seed & 0xFFFFFFFF, seed >> 32])
        assert orc.draw(seed, tag, chain, t, row, col) == int(out[col & 3])


def test_beta_schedule():
    for t, key in [(0, "beta_t0"), (249, "beta_t249"), (250, "beta_t250"), (999, "beta_t999")]:
        assert orc.beta_at(1.25, 0.25, 250, t) == GV[key]


@pytest.mark.parametrize("beta,key", [(1.0, "score_diff_beta1"), (2.0, "score_diff_beta2")])
def test_paper_score_difference(beta, key):
    """interior site, 8 neighbours at level 1, g = 1, l = 2, J = 1/3,
    sigma = 0.25: log p(1)/p(0) = 2 beta J 8 + 1/(2 sigma^2) (q = 0).  The inertia term
    subtracts beta*q from every label other than the current one."""
    m = orc.model(3, 3, 2, nbhd=8, periodic=False, J=GV["J_paper"], q=0.0, sigma=0.25)
    x = np.ones((3, 3), np.uint8)
    g = np.ones((3, 3), np.uint8)
    p = orc.pca_site_probs(m, x, g, 1, 1, beta)
    assert math.log(p[1] / p[0]) == pytest.approx(GV[key], rel=1e-13)
    m.q = GV["q_paper"]
    p = orc.pca_site_probs(m, x, g, 1, 1, beta)  # x_i = 1: label 0 pays c = beta q
    assert math.log(p[1] / p[0]) == pytest.approx(GV[key] + beta * GV["q_paper"], rel=1e-13)
    x[1, 1] = 0  # x_i = 0: label 1 pays c
    p = orc.pca_site_probs(m, x, g, 1, 1, beta)
    assert math.log(p[1] / p[0]) == pytest.approx(GV[key] - beta * GV["q_paper"], rel=1e-13)


CASES = [
    dict(H=3, W=3, levels=2, nbhd=4, periodic=True),
    dict(H=3, W=3, levels=2, nbhd=8, periodic=True),
    dict(H=3, W=4, levels=2, nbhd=8, periodic=False),
    dict(H=2, W=2, levels=3, nbhd=8, periodic=False),
    dict(H=1, W=3, levels=4, nbhd=8, periodic=False),
    dict(H=4, W=3, levels=5, nbhd=4, periodic=False),
    dict(H=3, W=5, levels=9, nbhd=8, periodic=True),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("pexp", [0, 1, 2])
def test_site_laws_match_enumeration(case, pexp):
    """C per-site PCA and Gibbs conditionals == enumerate.site_laws (independent code), for
    the L0 inertia of the paper and the L1 / L2 alternatives."""
    rng = np.random.default_rng(7)
    lat = en.Lattice(case["H"], case["W"], case["levels"], case["nbhd"], case["periodic"])
    m = orc.model(**case, J=1 / 3, q=0.51, sigma=0.3, inertia_p=pexp)
    for beta in (0.7, 1.25, 2.0):
        x = rng.integers(0, case["levels"], (case["H"], case["W"]), dtype=np.uint8)
        g = rng.integers(0, case["levels"], (case["H"], case["W"]), dtype=np.uint8)
        a, b, c = en.coefficients(beta, 1 / 3, 0.51, 0.3)
        ref = en.site_laws(lat, x.reshape(-1), g.reshape(-1), a, b, c, p=pexp)
        refg = en.site_laws(lat, x.reshape(-1), g.reshape(-1), a, b, c, inertia=False)
        for r in range(case["H"]):
            for cc in range(case["W"]):
                i = r * case["W"] + cc
                assert np.abs(orc.pca_site_probs(m, x, g, r, cc, beta) - ref[i]).max() < 1e-14
                assert np.abs(orc.gibbs_site_probs(m, x, g, r, cc, beta) - refg[i]).max() < 1e-14


def test_decide_inverse_cdf():
    """min{k < l-1: u < F_k} else l-1 over ascending labels, margin = min |u - F_k|."""
    p = np.array([0.25, 0.5, 0.25])
    assert orc.decide(p, 0.0) == (0, 0.25)
    assert orc.decide(p, 0.2499)[0] == 0
    assert orc.decide(p, 0.25)[0] == 1  # u == F_0 is not < F_0
    assert orc.decide(p, 0.7499)[0] == 1
    assert orc.decide(p, 0.75)[0] == 2
    w, mg = orc.decide(p, 0.9)
    assert w == 2 and mg == pytest.approx(0.15)


def _chi2_ok(counts, probs, n):
    """Pearson chi-square with expected >= 5 cells pooled; accept at ~1e-4 level."""
    e = probs * n
    keep = e >= 5
    obs = np.append(counts[keep], counts[~keep].sum())
    exp = np.append(e[keep], e[~keep].sum())
    if exp[-1] == 0:
        obs, exp = obs[:-1], exp[:-1]
    stat = ((obs - exp) ** 2 / exp).sum()
    dof = len(obs) - 1
    # Wilson-Hilferty upper quantile for p = 1e-4 (z = 3.72)
    crit = dof * (1 - 2 / (9 * dof) + 3.72 * math.sqrt(2 / (9 * dof))) ** 3
    return stat < crit, stat, crit


def test_one_step_frequencies_match_transition_matrix():
    """The C sweep's empirical one-step law from a fixed x equals the row P(x, .) of the
    exact transition matrix, over independent streams (chain ids)."""
    lat = en.Lattice(2, 2, 2, nbhd=8, periodic=False)
    m = orc.model(2, 2, 2, nbhd=8, periodic=False, J=1 / 3, q=0.51, sigma=0.5)
    g = np.array([[0, 1], [1, 1]], np.uint8)
    x = np.array([[1, 0], [0, 1]], np.uint8)
    beta = 1.25
    a, b, c = en.coefficients(beta, 1 / 3, 0.51, 0.5)
    P = en.pca_matrix(lat, g.reshape(-1), a, b, c)
    row = P[en.state_index(lat, x.reshape(-1))]
    n = 40000
    counts = np.zeros(16)
    for k in range(n):
        w, _ = orc.pca_sweep(m, x, g, beta, seed=99, chain=k, t=5)
        counts[en.state_index(lat, w.reshape(-1))] += 1
    ok, stat, crit = _chi2_ok(counts, row, n)
    assert ok, (stat, crit)


def _histogram(run_step, lat, x0, n_burn, n):
    x = x0.copy()
    counts = np.zeros(lat.levels ** lat.n)
    for t in range(n_burn + n):
        x = run_step(x, t)
        if t >= n_burn:
            counts[en.state_index(lat, x.reshape(-1))] += 1
    return counts / n


def test_pca_chain_reaches_closed_form_stationary_law():
    """Long C PCA chain on a 2x2 Moore lattice: empirical law -> pi~ (PAPER.md:250-255,
    closed form with R2), and clearly not pi_GS(a, b)."""
    lat = en.Lattice(2, 2, 2, nbhd=8, periodic=False)
    m = orc.model(2, 2, 2, nbhd=8, periodic=False, J=1 / 3, q=0.51, sigma=0.5)
    g = np.array([[0, 1], [1, 1]], np.uint8)
    beta = 1.25
    a, b, c = en.coefficients(beta, 1 / 3, 0.51, 0.5)
    cf = en.pca_closed_form(lat, g.reshape(-1), a, b, c)
    gs = en.gibbs_posterior(lat, g.reshape(-1), a, b)
    emp = _histogram(lambda x, t: orc.pca_sweep(m, x, g, beta, 5, 0, t)[0], lat,
                     g.copy(), 100, 60000)
    assert en.tv(emp, cf) < 0.015
    assert en.tv(cf, gs) > 0.05


def test_gibbs_chain_reaches_posterior():
    """Long C systematic-Gibbs chain: empirical law -> pi_GS(a, b)."""
    lat = en.Lattice(2, 2, 3, nbhd=8, periodic=False)
    m = orc.model(2, 2, 3, nbhd=8, periodic=False, J=1 / 3, q=0.0, sigma=0.5)
    g = np.array([[0, 2], [1, 2]], np.uint8)
    beta = 1.0
    a, b, _ = en.coefficients(beta, 1 / 3, 0.0, 0.5)
    gs = en.gibbs_posterior(lat, g.reshape(-1), a, b)
    emp = _histogram(lambda x, t: orc.gibbs_sweep(m, x, g, beta, 11, 0, t), lat, g.copy(), 100,
                     60000)
    assert en.tv(emp, gs) < 0.02


def test_q0_single_site_equals_gibbs_and_large_q_freezes():
    """q = 0 on a 1x1 lattice the PCA and Gibbs laws coincide; q -> inf
    freezes the chain."""
    m = orc.model(1, 1, 5, q=0.0, sigma=0.25)
    x = np.array([[3]], np.uint8)
    g = np.array([[1]], np.uint8)
    assert np.array_equal(orc.pca_site_probs(m, x, g, 0, 0, 1.5), orc.gibbs_site_probs(m, x, g, 0, 0, 1.5))
    rng = np.random.default_rng(1)
    m = orc.model(16, 16, 5, q=1e6, sigma=0.25)
    x = rng.integers(0, 5, (16, 16), dtype=np.uint8)
    g = rng.integers(0, 5, (16, 16), dtype=np.uint8)
    w, _ = orc.pca_sweep(m, x, g, 1.25, 1, 0, 0)
    assert np.array_equal(w, x)


def test_mpm_counts_and_ties():
    """MPM (R15): argmax of counts, ties to the lowest label; counts cover every sweep
    t >= burn_in exactly once per site."""
    counts = np.array([[[3, 2, 1]], [[3, 4, 1]], [[0, 0, 2]]], np.uint32)
    assert orc.mpm(counts).tolist() == [[0, 1, 2]]
    m = orc.model(6, 7, 3, nbhd=8, periodic=False, sigma=0.4)
    rng = np.random.default_rng(3)
    g = rng.integers(0, 3, (6, 7), dtype=np.uint8)
    x, cnt = orc.pca_run(m, g, g, 30, 1.25, 0.25, 10, seed=4, burn_in=12)
    assert (cnt.sum(axis=0) == 18).all()
    x2, _ = orc.pca_run(m, g, g, 30, 1.25, 0.25, 10, seed=4, burn_in=-1)
    assert np.array_equal(x, x2)
    # splitting a run preserves the chain (RNG keyed by the global sweep index)
    xa, ca = orc.pca_run(m, g, g, 17, 1.25, 0.25, 10, seed=4, burn_in=12)
    xb, cb = orc.pca_run(m, xa, g, 13, 1.25, 0.25, 10, seed=4, t0=17, burn_in=12)
    assert np.array_equal(xb, x) and np.array_equal(ca + cb, cnt)


def test_metrics_special_cases():
    """PAPER.md:516-534 with R16/R17: MSE on luminance, PSNR with the ORIGINAL's max,
    global SSIM with c1 = 1e-4, c2 = 9e-4."""
    # luminances (0,0) vs (1,0) -> 0.5
    mse, psnr, ssim, st = orc.metrics(np.array([[0], [0]]), np.array([[1], [0]]), 2)
    assert mse == 0.5 and st == -1  # original all black: PSNR undefined
    # PSNR = 20 dB at max 1 and MSE 0.01 (l = 11: one level = 0.1)
    x = np.array([[10, 0, 5, 7]], np.uint8)
    y = np.array([[9, 1, 4, 8]], np.uint8)
    mse, psnr, ssim, st = orc.metrics(x, y, 11)
    assert mse == pytest.approx(0.01, rel=1e-14) and psnr == pytest.approx(GV["psnr_mse_0p01"], abs=1e-12)
    # PSNR at MSE 0.0025: l = 21 (step 0.05), every pixel one level off
    x = np.array([[20, 3, 4, 9]], np.uint8)
    y = np.array([[19, 4, 3, 10]], np.uint8)
    _, psnr, _, _ = orc.metrics(x, y, 21)
    assert psnr == pytest.approx(GV["psnr_mse_0p0025"], abs=1e-11)
    # x == y: MSE 0, PSNR inf, SSIM 1
    rng = np.random.default_rng(0)
    z = rng.integers(0, 9, (16, 16), dtype=np.uint8)
    mse, psnr, ssim, _ = orc.metrics(z, z, 9)
    assert mse == 0 and psnr == math.inf and ssim == pytest.approx(1.0, abs=1e-15)
    # two constant images a != b: (2ab + c1)/(a^2 + b^2 + c1)
    a, b = 0.25, 0.75
    _, _, ssim, _ = orc.metrics(np.full((4, 4), 1, np.uint8), np.full((4, 4), 3, np.uint8), 5)
    assert ssim == pytest.approx((2 * a * b + 1e-4) / (a * a + b * b + 1e-4), rel=1e-14)
    # symmetry and a naive recomputation from moments
    w = rng.integers(0, 9, (16, 16), dtype=np.uint8)
    _, _, s1, _ = orc.metrics(z, w, 9)
    _, _, s2, _ = orc.metrics(w, z, 9)
    assert s1 == pytest.approx(s2, abs=1e-15)
    lx, ly = z / 8.0, w / 8.0
    cov = ((lx - lx.mean()) * (ly - ly.mean())).mean()
    ref = ((2 * lx.mean() * ly.mean() + 1e-4) * (2 * cov + 9e-4)) / (
        (lx.mean() ** 2 + ly.mean() ** 2 + 1e-4) * (lx.var() + ly.var() + 9e-4))
    assert s1 == pytest.approx(ref, abs=1e-13)


def test_windowed_ssim_properties():
    rng = np.random.default_rng(5)
    z = rng.integers(0, 5, (20, 23), dtype=np.uint8)
    assert orc.ssim_windowed(z, z, 5) == pytest.approx(1.0, abs=1e-14)
    w = z.copy()
    w[10, 10] = (w[10, 10] + 2) % 5
    s = orc.ssim_windowed(z, w, 5)
    assert 0.5 < s < 1.0
    # one 7x7 image = one window: equals the global SSIM with sample covariance
    a = rng.integers(0, 5, (7, 7), dtype=np.uint8)
    b = rng.integers(0, 5, (7, 7), dtype=np.uint8)
    la, lb = a / 4.0, b / 4.0
    cov = ((la - la.mean()) * (lb - lb.mean())).sum() / 48
    ref = ((2 * la.mean() * lb.mean() + 1e-4) * (2 * cov + 9e-4)) / (
        (la.mean() ** 2 + lb.mean() ** 2 + 1e-4) * (la.var(ddof=1) + lb.var(ddof=1) + 9e-4))
    assert orc.ssim_windowed(a, b, 5) == pytest.approx(ref, abs=1e-13)
    # a change at the corner pixel touches only the window at (0, 0): the mean over the
    # (H-6)(W-6) stride-1 windows is (count - 1 + SSIM_window(0,0)) / count
    def one(wa, wb):
        la, lb = wa / 4.0, wb / 4.0
        cv = ((la - la.mean()) * (lb - lb.mean())).sum() / 48
        return ((2 * la.mean() * lb.mean() + 1e-4) * (2 * cv + 9e-4)) / (
            (la.mean() ** 2 + lb.mean() ** 2 + 1e-4) * (la.var(ddof=1) + lb.var(ddof=1) + 9e-4))
    c = z.copy()
    c[0, 0] = (c[0, 0] + 3) % 5
    count = (20 - 6) * (23 - 6)
    assert orc.ssim_windowed(z, c, 5) == pytest.approx((count - 1 + one(z[:7, :7], c[:7, :7])) / count,
                                                        abs=1e-13)


def test_quantizer():
    """l = 5, 0.5 + 0.13 = 0.63 -> level 3; ties go to the lower level (R12)."""
    assert orc.quantize(0.63, 5) == 3
    assert orc.quantize(0.125, 5) == 0
    assert orc.quantize(0.1250001, 5) == 1
    assert orc.quantize(1.0, 5) == 4 and orc.quantize(0.0, 33) == 0


@pytest.mark.parametrize("levels,sigma,level,expected", [
    (5, 0.25, 2, math.erf(0.125 / (0.25 * math.sqrt(2)))),            # 0.3829
    (5, 0.25, 0, 0.5 + 0.5 * math.erf(0.125 / (0.25 * math.sqrt(2)))),  # 0.6915: clamped edge
    (9, 0.20, 4, math.erf(0.0625 / (0.2 * math.sqrt(2)))),            # 0.2453
    (33, 0.10, 16, math.erf(0.015625 / (0.1 * math.sqrt(2)))),        # 0.1242
])
def test_degrade_unchanged_fraction(levels, sigma, level, expected):
    """add N(0, sigma^2), clamp, round to nearest level.  On a constant
    image the unchanged fraction is P(|eps| < half a level gap) (Gaussian CDF)."""
    x = np.full((256, 256), level, np.uint8)
    y = orc.degrade(x, levels, sigma, seed=17)
    assert y.max() < levels
    assert abs((y == x).mean() - expected) < 0.01


def test_degrade_tiny_noise_is_identity_and_gauss_moments():
    rng = np.random.default_rng(2)
    x = rng.integers(0, 9, (32, 32), dtype=np.uint8)
    assert np.array_equal(orc.degrade(x, 9, 1e-12, seed=3), x)
    z = np.array([orc.gauss(8, 0, r, c) for r in range(200) for c in range(250)])
    assert abs(z.mean()) < 4 / math.sqrt(len(z))
    assert abs(z.var() - 1) < 0.03


def test_generate_mrf():
    """uniform random start, then prior-only Gibbs.  Zero sweeps =
    i.i.d. uniform labels; a cold long run orders the lattice."""
    m = orc.model(64, 64, 4, nbhd=8)
    x = orc.generate_mrf(m, 0, 1.0, 1.0, seed=5)
    ok, stat, crit = _chi2_ok(np.bincount(x.reshape(-1), minlength=4).astype(float),
                              np.full(4, 0.25), x.size)
    assert ok
    # the prior "favors configurations where pixels are aligned with their
    # neighbors": after a cold run almost every neighbour pair agrees (random start: 1/2).
    m = orc.model(16, 16, 2, nbhd=8)
    for s in range(5):
        y = orc.generate_mrf(m, 100, 0.5, 50.0, seed=s).astype(int)
        agree = np.concatenate([(y[1:, :] == y[:-1, :]).ravel(), (y[:, 1:] == y[:, :-1]).ravel(),
                                (y[1:, 1:] == y[:-1, :-1]).ravel(), (y[1:, :-1] == y[:-1, 1:]).ravel()])
        assert agree.mean() > 0.9


# --- checkerboard-colour Gibbs scan (the GPU Gibbs sampler's order) ---

@pytest.mark.parametrize("lat", [en.Lattice(4, 6, 2, nbhd=4, periodic=True),
                                 en.Lattice(4, 6, 2, nbhd=8, periodic=True),
                                 en.Lattice(3, 5, 2, nbhd=8, periodic=False),
                                 en.Lattice(5, 3, 2, nbhd=4, periodic=False)])
def test_gibbs_colours_are_independent_sets(lat):
    """No two sites of one colour are neighbours (even torus sides; any free lattice), so a
    colour class may be updated at once (checked on the enumeration's own neighbour lists)."""
    nbrs = lat.neighbours()
    col = [orc.gibbs_colour(lat.nbhd, i // lat.W, i % lat.W) for i in range(lat.n)]
    assert len(set(col)) == (2 if lat.nbhd == 4 else 4)
    for i in range(lat.n):
        for j in nbrs[i]:
            assert col[i] != col[j]


def test_coloured_sweep_is_any_order_within_a_colour():
    """Updating the sites of one colour in a random order, one at a time from the current
    state (site conditional of PAPER.md:417-429, tag GIBBS uniform), gives exactly the
    coloured sweep: the sites of a colour do not see each other."""
    H, W, L = 6, 8, 5
    m = orc.model(H, W, L, nbhd=8, periodic=True, J=1 / 3, q=0.0, sigma=0.3)
    rng = np.random.default_rng(3)
    g = rng.integers(0, L, (H, W)).astype(np.uint8)
    x = rng.integers(0, L, (H, W)).astype(np.uint8)
    beta, seed, chain, t = 1.4, 17, 2, 9
    ref = orc.gibbs_sweep_coloured(m, x, g, beta, seed, chain, t)
    y = x.copy()
    for k in range(4):
        sites = [(r, c) for r in range(H) for c in range(W) if orc.gibbs_colour(8, r, c) == k]
        for idx in rng.permutation(len(sites)):
            r, c = sites[idx]
            p = orc.gibbs_site_probs(m, y, g, r, c, beta)
            u = orc.draw(seed, 2, chain, t, r, c) / 2.0 ** 32
            y[r, c] = orc.decide(p, u)[0]
    assert np.array_equal(y, ref)
    assert not np.array_equal(ref, orc.gibbs_sweep(m, x, g, beta, seed, chain, t))  # != column scan


@pytest.mark.parametrize("lat,g", [(en.Lattice(2, 3, 2, nbhd=4), np.array([[0, 1, 1], [1, 0, 1]])),
                                   (en.Lattice(2, 3, 3, nbhd=8), np.array([[0, 2, 1], [2, 2, 0]]))])
def test_coloured_sweep_law_is_the_product_of_site_kernels(lat, g):
    """The C coloured sweep's one-step law from a fixed x equals the row of
    K_{i1} K_{i2} ... K_{in} (sites in colour order), the single-site Gibbs kernels of the
    enumeration (independent code), over independent streams (chain ids)."""
    m = orc.model(lat.H, lat.W, lat.levels, nbhd=lat.nbhd, periodic=False, J=1 / 3, q=0.0,
                  sigma=0.5)
    g = g.astype(np.uint8)
    beta = 1.25
    a, b, _ = en.coefficients(beta, 1 / 3, 0.0, 0.5)
    order = sorted(range(lat.n), key=lambda i: (orc.gibbs_colour(lat.nbhd, i // lat.W, i % lat.W), i))
    K = np.eye(lat.levels ** lat.n)
    for i in order:
        K = K @ en.gibbs_site_kernel(lat, g.reshape(-1), a, b, i)
    x = np.array([[1, 0, 1], [0, 1, 1]], np.uint8) % lat.levels
    row = K[en.state_index(lat, x.reshape(-1))]
    n = 30000
    counts = np.zeros(len(row))
    for k in range(n):
        w = orc.gibbs_sweep_coloured(m, x, g, beta, seed=5, chain=k, t=3)
        counts[en.state_index(lat, w.reshape(-1))] += 1
    ok, stat, crit = _chi2_ok(counts, row, n)
    assert ok, (stat, crit)
    gs = en.gibbs_posterior(lat, g.reshape(-1), a, b)
    assert np.abs(gs @ K - gs).max() < 1e-15  # the coloured sweep leaves pi_GS invariant


def _site_kernel_product(lat, g, a, b, order):
    K = np.eye(lat.levels ** lat.n)
    for i in order:
        K = K @ en.gibbs_site_kernel(lat, g.reshape(-1), a, b, i)
    return K


@pytest.mark.parametrize("lat,g", [(en.Lattice(2, 3, 2, nbhd=8), np.array([[0, 1, 1], [1, 0, 1]])),
                                   (en.Lattice(3, 2, 2, nbhd=8), np.array([[0, 1], [1, 1], [0, 0]])),
                                   (en.Lattice(2, 2, 3, nbhd=8), np.array([[0, 2], [1, 2]]))])
def test_column_major_sweep_law_is_the_product_of_site_kernels(lat, g):
    """The paper's systematic scan (section 5.1: pixels visited column by
    column, R13): the C sweep's one-step law from a fixed x equals the row of
    K_{i1} ... K_{in} with the sites in COLUMN-MAJOR order (c outer, r inner), built from the
    enumeration's single-site Gibbs kernels (independent code).  The same frequencies must
    reject the row-major product, so a scan in the wrong order fails this pin.  Moore-8 only:
    on the 4-neighbour grid both scans orient every edge from (r, c) towards larger r or c,
    so they are linear extensions of the same order and have the SAME law (checked below);
    the anti-diagonal Moore edges (r, c+1)-(r+1, c) are oriented oppositely by the two."""
    m = orc.model(lat.H, lat.W, lat.levels, nbhd=lat.nbhd, periodic=False, J=1 / 3, q=0.0,
                  sigma=0.5)
    g = g.astype(np.uint8)
    beta = 1.25
    a, b, _ = en.coefficients(beta, 1 / 3, 0.0, 0.5)
    col_major = sorted(range(lat.n), key=lambda i: (i % lat.W, i // lat.W))
    row_major = list(range(lat.n))
    x = (np.arange(lat.n).reshape(lat.H, lat.W) % 2).astype(np.uint8)
    k_col = _site_kernel_product(lat, g, a, b, col_major)[en.state_index(lat, x.reshape(-1))]
    k_row = _site_kernel_product(lat, g, a, b, row_major)[en.state_index(lat, x.reshape(-1))]
    assert 0.5 * np.abs(k_col - k_row).sum() > 0.02  # the two scan orders have different laws
    lat4 = en.Lattice(lat.H, lat.W, lat.levels, nbhd=4)
    k4 = [_site_kernel_product(lat4, g, a, b, o)[en.state_index(lat4, x.reshape(-1))]
          for o in (col_major, row_major)]
    assert np.abs(k4[0] - k4[1]).max() < 1e-15  # 4-neighbour: indistinguishable orders
    n = 30000
    counts = np.zeros(len(k_col))
    for k in range(n):
        w = orc.gibbs_sweep(m, x, g, beta, seed=6, chain=k, t=4)
        counts[en.state_index(lat, w.reshape(-1))] += 1
    ok, stat, crit = _chi2_ok(counts, k_col, n)
    assert ok, (stat, crit)
    bad, stat_row, _ = _chi2_ok(counts, k_row, n)
    assert not bad, stat_row


def test_coloured_gibbs_run_counts():
    """orc_gibbs_run(order = colour) == repeated coloured sweeps, with counts of x after
    every sweep t >= burn_in."""
    m = orc.model(6, 8, 3, nbhd=4, periodic=True, J=1 / 3, q=0.0, sigma=0.4)
    rng = np.random.default_rng(8)
    g = rng.integers(0, 3, (6, 8)).astype(np.uint8)
    x, cnt = orc.gibbs_run(m, g, g, 12, 1.0, 0.5, 4, 21, chain=1, burn_in=5, order="colour")
    y = g.copy()
    ref = np.zeros_like(cnt)
    for t in range(12):
        y = orc.gibbs_sweep_coloured(m, y, g, orc.beta_at(1.0, 0.5, 4, t), 21, 1, t)
        if t >= 5:
            for k in range(3):
                ref[k] += (y == k)
    assert np.array_equal(x, y) and np.array_equal(cnt, ref)


def test_windowed_ssim_against_filter_implementation():
    """orc_ssim_windowed (explicit 7x7 loops) against an independent filter formulation:
    window means and sample (co)variances from scipy.ndimage.uniform_filter over the valid
    window centres, then the mean of the SSIM map (Wang et al.'s definition, R16)."""
    from scipy.ndimage import uniform_filter

    rng = np.random.default_rng(12)
    for L, shape in [(5, (23, 31)), (2, (7, 40)), (33, (16, 16))]:
        x = rng.integers(0, L, shape).astype(np.uint8)
        y = np.clip(x.astype(int) + rng.integers(-1, 2, shape), 0, L - 1).astype(np.uint8)
        a, b = x / (L - 1.0), y / (L - 1.0)
        n = 49.0
        f = lambda z: uniform_filter(z, size=7, mode="constant")[3:-3, 3:-3]  # valid centres
        mx, my = f(a), f(b)
        vx = (f(a * a) - mx * mx) * n / (n - 1)
        vy = (f(b * b) - my * my) * n / (n - 1)
        cxy = (f(a * b) - mx * my) * n / (n - 1)
        ssim_map = ((2 * mx * my + 1e-4) * (2 * cxy + 9e-4)) / ((mx ** 2 + my ** 2 + 1e-4) * (vx + vy + 9e-4))
        assert orc.ssim_windowed(x, y, L) == pytest.approx(float(ssim_map.mean()), abs=1e-12)
