"""Pins for the Zirr & Kaplanyan-style baseline of the oracle (eval_mode 3,
DESIGN.md §10, readings R-31..R-36): footprint probes vs the
SVD of the Jacobian, the area-quadrupling LOD pair vs Eq. 7's expectation, the
classical binomial of Eq. 15 vs the exact Bernoulli-sum law and
vs the Gaussian written out with scipy's normal quantiles, and the whole
path's expectation vs the smooth microfacet BRDF (Eq. 5-6)."""
import math

import numpy as np
import pytest
from scipy import stats as st

from oracle import stats


def _J(P, r, th):
    smax, smin = math.sqrt(P * r), math.sqrt(P / r)
    c, s = math.cos(th), math.sin(th)
    J = np.array([[c, -s], [s, c]]) @ np.diag([smax, smin])
    return J.astype(np.float32).astype(np.float64)


def test_zk_probes_vs_svd(orc):
    """n = min(ceil(s1/s2), 16) probes of area P/n, centred on the line through
    (u, v) along the major singular vector, symmetric, spaced s1/n (P:L188,
    L1087; R-31/R-32)."""
    rng = np.random.default_rng(31)
    for _ in range(3000):
        J = _J(2.0 ** rng.uniform(-30, 0), 2.0 ** rng.uniform(0, 6.5), rng.uniform(0, math.pi))
        U, S, _ = np.linalg.svd(J)
        u0, v0 = (float(np.float32(x)) for x in rng.uniform(-100, 100, 2))
        n, uk, vk, A, fl = orc.zk_probes([J[0, 0], J[1, 0], J[0, 1], J[1, 1]], u0, v0)
        r = S[0] / S[1]
        if abs(r - round(r)) < 1e-4 * r:
            continue                                  # ceil() at a rounding boundary
        assert n == min(math.ceil(r), 16)
        assert (fl == 4) == (math.ceil(r) > 16)
        assert abs(A * n - S[0] * S[1]) <= 2e-6 * S[0] * S[1]
        pts = np.stack([np.array(uk) - u0, np.array(vk) - v0], 1)
        e = U[:, 0]
        along = pts @ e
        across = pts @ np.array([-e[1], e[0]])
        tol = 1e-5 * S[0] + 2.5e-7 * (abs(u0) + abs(v0))           # fp32 rounding of uv + offset
        assert np.all(np.abs(across) <= tol)
        assert np.all(np.abs(along + along[::-1]) <= 2 * tol)        # symmetric about (u, v)
        if n > 1:
            sp = np.diff(along) * np.sign(along[-1] - along[0])
            assert np.all(np.abs(sp - S[0] / n) <= 1e-4 * S[0] / n + 2 * tol)


def test_zk_isotropic_single_probe(orc):
    n, uk, vk, A, fl = orc.zk_probes([1 / 64, 0, 0, 1 / 64], 0.25, 0.75)
    assert n == 1 and uk == [0.25] and vk == [0.75] and A == 2.0 ** -12 and fl == 0


def test_zk_lod_pair_conserves_area(orc):
    """Cells quadruple in area per level; the output mix weight t/3 on
    the top level makes (1 - t/3) 4^kz + (t/3) 4^(kz+1) = A (Eq. 7, R-33)."""
    rng = np.random.default_rng(33)
    for A in np.float32(2.0 ** rng.uniform(-70, 40, 5000)):
        kz, t = orc.zk_lod(float(A))
        assert 0.0 <= t < 3.0
        assert abs((1 - t / 3) * 4.0 ** kz + (t / 3) * 4.0 ** (kz + 1) - float(A)) <= 1e-6 * float(A)
    for k in (-20, -3, 0, 5):
        assert orc.zk_lod(4.0 ** k) == (k, 0.0)
        assert orc.zk_lod(2 * 4.0 ** k) == (k, 1.0)


@pytest.mark.parametrize("nt,p", [(1.0, 0.3), (4.0, 0.5), (6.25, 0.3), (16.0, 0.3), (1.5625, 0.9),
                                  (10.75, 0.05), (0.4, 0.7)])
def test_zk_count_looped_regime_is_the_bernoulli_sum(orc, nt, p):
    """n p <= 5 and n <= 16: the sum of floor(n) Bernoulli trials plus one
    fractional trial (Eq. 15 lower branch, R-35): its law is Bin(floor n, p) *
    Bernoulli(frac(n) p), with p quantised up to 2^-24."""
    rng = np.random.default_rng(int(nt * 100 + p * 10))
    ws = rng.integers(0, 2 ** 32, 40000, dtype=np.uint64)
    c = np.array([orc.zk_count(int(w), nt, p) for w in ws], dtype=np.int64)
    nf = int(math.floor(nt))
    pq = math.ceil(np.float32(p) * 2 ** 24) / 2 ** 24
    pf = math.ceil(float(np.float32(np.float32(nt - nf) * np.float32(p))) * 2 ** 24) / 2 ** 24
    law = np.convolve(st.binom.pmf(np.arange(nf + 1), nf, pq), [1 - pf, pf])
    assert c.min() >= 0 and c.max() <= nf + 1
    assert stats.chi2_gof(np.bincount(c, minlength=len(law)), law) > 1e-3
    assert abs(c.mean() - nt * p) < 4 * math.sqrt(nt * p * (1 - p) / len(c)) + 1e-6


def test_zk_count_special_cases(orc):
    for w in (0, 12345, 2 ** 32 - 1):
        assert orc.zk_count(w, 7.0, 0.0) == 0
        assert orc.zk_count(w, 5.0, 1.0) == 5            # looped: every trial succeeds
        assert orc.zk_count(w, 0.0, 0.5) == 0
        assert orc.zk_count(w, 40.0, 1.0) == 40          # Gaussian: sigma = 0, mu = n


@pytest.mark.parametrize("nt,p", [(10.0, 0.6), (16.5, 0.1), (1000.0, 0.034), (64.0, 0.5), (2.0 ** 20, 0.2)])
def test_zk_count_gaussian_regime_matches_eq15(orc, nt, p):
    """n p > 5 or n > 16: floor(N(theta; mu = n p, sigma^2 = n p (1-p))) clamped
    to [0, ceil n] (Eq. 15 upper branch, R-34), theta quantised to the 4096
    quantile cells: every cell against scipy's normal quantile in fp64 (a cell
    may differ by one where mu + sigma z lands within fp32 rounding of an
    integer: about 2 ulp(mu + 4 sigma) of the cells)."""
    q = np.arange(4096)
    c = np.array([orc.zk_count(int(k) << 2, nt, p) for k in q])
    mu = nt * p
    sg = math.sqrt(mu * (1 - p))
    ref = np.floor(np.clip(mu + sg * st.norm.ppf((q + 0.5) / 4096), 0, math.ceil(nt)))
    d = c - ref
    ulp = float(np.spacing(np.float32(mu + 4 * sg)))
    assert np.all(np.abs(d) <= 1) and np.count_nonzero(d) <= 3 + 4096 * 4 * ulp
    # floor bias of the classical approximation: E = n p - 1/2 + O(clamp)
    if mu > 5 * max(1.0, sg) and sg > 1:
        assert abs(c.mean() - (mu - 0.5)) < 0.05


def _gbuf(duv, uv, N, alpha, R, objs):
    n = len(uv)
    return dict(duv=np.broadcast_to(np.asarray(duv, np.float32), (n, 4)).copy(),
                uvm=np.concatenate([uv.astype(np.float32), np.asarray(objs, np.uint32).view(np.float32)[:, None],
                                    np.ones((n, 1), np.uint32).view(np.float32)], 1),
                nrm=np.tile(np.array([0, 0, 1, 0], np.float32), (n, 1)), pos=np.zeros((n, 4), np.float32),
                mat=np.tile(np.array([alpha, alpha, N, R], np.float32), (n, 1)))


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
@pytest.mark.parametrize("r_foot", [1.0, 5.5])
def test_zk_expectation_is_the_smooth_brdf(orc, ndf, r_foot):
    """In the looped regime the counts are exact Bernoulli sums, so E[C] = N P p
    and the mean radiance over independent surface points (distinct object ids)
    equals the smooth microfacet radiance F G2 D(h) E / (4 n.wi) (Eq. 5-6)."""
    from paper_2306_05051_b200 import synth
    rng = np.random.default_rng(35)
    M = 3000
    P, alpha, R, N = 2.0 ** -5, 0.4, 0.3, 100.0
    J = _J(P, r_foot, 0.6)
    uv = rng.random((M, 2))
    g = _gbuf([J[0, 0], J[1, 0], J[0, 1], J[1, 1]], uv, N, alpha, R, rng.integers(0, 2 ** 31, M))
    s30 = math.sin(math.radians(30))
    wi, wo = (s30, 0.0, math.cos(math.radians(30))), (-s30, 0.0, math.cos(math.radians(30)))
    sc = synth.SceneParams(seed=3, ndf=ndf, view_kind="directional", view=wi,
                           lights=[synth.Light("directional", wo, (1.0, 1.0, 1.0))], method="zk")
    rgb, fl, _ = orc.eval(g, sc)
    assert np.all(fl == 0)
    h = np.array([0.0, 0.0, 1.0])
    D = float(stats.ndf_D(ndf, alpha, alpha, h[None])[0])
    cih = float(np.dot(wi, h))
    F = 0.9 + 0.1 * (1 - cih) ** 5
    wl = np.array(wi)
    G2 = orc.smith_g2(ndf, alpha, alpha, wl, np.array(wo))
    smooth = F * G2 * D / (4 * wl[2])
    x = rgb[:, 0]
    assert abs(x.mean() / smooth - 1) < 4 * x.std() / math.sqrt(M) / smooth + 1e-3
