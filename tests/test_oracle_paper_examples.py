"""Pins to values the paper prints (Fig. 4 worked example; the
48-draw budget) and to closed forms worked by hand for config C1."""
import math
import os

import numpy as np
import pytest

from oracle import stats

GOLD = os.path.join(os.path.dirname(__file__), "golden", "fig4_points.txt")


def _fig4():
    a = np.loadtxt(GOLD)
    return a[:, :2], a[:, 2].astype(int)


def test_fig4_printed_realization():
    """Fig. 4(a): 64 stratified trials, p = 1/2; 33 successes; the drawn
    windows [0,.5)^2 and [0,.75)^2 hold floor(N P) = 16 and 36 points (Eq. 9,
    stratified N(P) = floor(N P)) with 12 and 23 successes."""
    pts, succ = _fig4()
    assert len(pts) == 64 and succ.sum() == 33
    cells = set(map(tuple, np.floor(pts * 8).astype(int)))
    assert len(cells) == 64                                  # one point per 1/8 cell
    assert stats.spatialized_count(pts, succ, (0, 0, 0.5, 0.5)) == (16, 12)
    assert stats.spatialized_count(pts, succ, (0, 0, 0.75, 0.75)) == (36, 23)
    assert math.floor(64 * 0.25) == 16 and math.floor(64 * 0.5625) == 36


def test_fig4_distributing_vs_blending(orc):
    """Fig. 4(b,c) setting: N = 64, p = 1/2, footprint P = 0.375 between the LOD
    areas 0.25 and 0.5, M = 10^4. The oracle's lattice distributes P as n_i =
    w_i N 2^ls_i = (8, 16) and the distributed law b(8) + b(16) is Binomial(24);
    stratified spatialised trials in a 24-cell window agree with it, while
    Zirr's output blend (Eq. 7) is rejected with ~50 % variance deficit."""
    ls, lr, jo, w, _ = orc.lattice(0.375, 1.0, 0.0)
    n = sorted(round(wi * 64 * 2.0 ** a, 6) for wi, a in zip(w, ls) if wi > 0)
    assert n == [8.0, 16.0]
    rng = np.random.default_rng(44)
    M = 10000
    dist = rng.binomial(8, 0.5, M) + rng.binomial(16, 0.5, M)
    pv = stats.chi2_gof(np.bincount(dist), stats.binom_pmf(24, 0.5))
    assert pv > 0.01
    spat = np.empty(M, int)
    for m in range(M):
        pts = stats.stratified_points(8, rng)
        succ = rng.random(64) < 0.5
        spat[m] = stats.spatialized_count(pts, succ, (0, 0, 0.75, 0.5))[1]
    assert stats.chi2_two_sample(dist, spat) > 0.01
    zirr = 0.5 * rng.binomial(32, 0.5, M) + 0.5 * rng.binomial(16, 0.5, M)
    assert np.var(zirr) < 0.75 * 6.0 and abs(np.var(dist) - 6.0) < 0.6
    zirr_int = np.floor(zirr).astype(int)
    assert stats.chi2_gof(np.bincount(zirr_int), stats.binom_pmf(24, 0.5)) < 0.01


def _c1(orc, ndf, variant):
    from paper_2306_05051_b200 import synth
    fr = synth.c1(ndf, variant)
    return orc.eval(fr.gbuf, fr.scene, debug=True)


def test_c1_mirror_worked_example(orc):
    """C1 mirror (h = n): P = 2^-12, one grid, n = 1e5 * 2^-12 = 24.4140625,
    p = R = 0.034, P>=1 = 1 - 0.966^n = 0.5702354, mu = 0.7960782,
    sigma = 0.8769330, cap = 25; angular g = (-1/2, -1/2) -> base node (-1,-1)."""
    rgb, fl, rec = _c1(orc, "ggx", "mirror")
    r = rec[:, 0]
    n = 1e5 * 2.0 ** -12
    assert np.all(r["P"] == 2.0 ** -12) and np.all(r["r"] == 1.0)
    assert np.all(r["n"][:, 0] == np.float32(n)) and np.all(r["n"][:, 1:] == 0)
    assert np.all(np.abs(r["p"] - 0.034) < 1e-8)
    pge1 = 1 - (1 - 0.034) ** n
    assert abs(pge1 - 0.5702354) < 1e-6
    assert np.all(np.abs(r["T"][:, 0] / 2 ** 23 - pge1) < 2 ** -22)
    assert np.all(np.abs(r["sigma"][:, 0] - math.sqrt((n - 1) * 0.034 * 0.966)) < 1e-6)
    assert np.all(np.abs(r["m1"][:, 0] - (1 + (n - 1) * 0.034)) < 1e-6)
    assert np.all(r["cap"][:, 0] == 25.0)
    assert np.all(r["cx0"] == -1) and np.all(r["cy0"] == -1)
    # only the first grid draws; the other three carry n = 0 -> count 0
    assert np.all(r["count"][:, 12:] == 0)
    # mean blended count vs the law's mean (enumerated), SURVEY: 0.8548
    pmf, _ = stats.gated_pmf_enumerated(float(np.float32(n)), float(np.float32(0.034)))
    assert abs(stats.pmf_mean(pmf) - 0.8548) < 2e-3
    assert abs(r["C"].mean() - stats.pmf_mean(pmf)) < 0.04
    assert np.all(fl == 0)


@pytest.mark.parametrize("ndf,ratio", [("ggx", 0.167355), ("beckmann", 0.213621)])
def test_c1_azimuth90_worked_example(orc, ndf, ratio):
    """C1b: h = (0.2672612, 0.2672612, 0.9258201), theta_h = 22.21 deg; with
    alpha = 0.3 the NDF ratio D(h)/D(n) is 0.167355 (GGX) / 0.213621
    (Beckmann); g = h_xy / 0.05 - 1/2 = 4.845 -> base node (4, 4)."""
    hx = 0.5 / math.sqrt(3.5)
    hz = math.sqrt(3.0) / math.sqrt(3.5)
    X2 = 2 * (hx / 0.3) ** 2
    ref = 1 / (X2 + hz * hz) ** 2 if ndf == "ggx" else math.exp(-X2 / hz ** 2) / hz ** 4
    assert abs(ref - ratio) < 1e-6
    rgb, fl, rec = _c1(orc, ndf, "az90")
    r = rec[:, 0]
    assert np.all(np.abs(r["p"] / 0.034 - ratio) < 2e-6)
    assert np.all(r["cx0"] == 4) and np.all(r["cy0"] == 4)
    pge1 = 1 - (1 - 0.034 * ratio) ** (1e5 * 2.0 ** -12)
    assert np.all(np.abs(r["T"][:, 0] / 2 ** 23 - pge1) < 2e-6)


def test_48_draws_per_pixel_light(orc):
    """4 grids x 3 simplex texels x 4 angular nodes = 48 draws, for
    any footprint: every active record carries 48 distinct draw hashes when
    its 4 grids are distinct."""
    from paper_2306_05051_b200 import synth
    gb = synth.random_gbuffer(16, 16, seed=5)
    sc = synth.random_scene(5, n_lights=2)
    _, fl, rec = orc.eval(gb, sc, debug=True)
    n_full = 0
    for r in rec.ravel():
        if not r["light_active"]:
            continue
        keys = {(a, b, c) for a, b, c in zip(r["ls"], r["lr"], r["jo"])}
        if len(keys) == 4:
            assert len(set(r["hash"].tolist())) == 48
            n_full += 1
    assert n_full > 50
