"""The oracle's own four checks (BASELINE.json north star), on tiny inputs:
1. brute force: explicit stratified facets with NDF-distributed normals,
   counted inside the footprint and a reflection cone, vs the distributed law
   built from the oracle's lattice (Eq. 10/13);
2. expected count = N P p (Eq. 3-4; P:L162 footnote);
3. convergence to the smooth NDF as density grows (Eq. 5-6, Fig. 13);
4. coherence between consecutive LODs."""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import stats


def _gbuf(duv, uv, N, ax, ay, R, obj=0):
    n = len(uv)
    duv = np.broadcast_to(np.asarray(duv, np.float32), (n, 4)).copy()
    uvm = np.zeros((n, 4), np.float32)
    uvm[:, :2] = uv
    uvm[:, 2] = np.array([obj] * n, np.uint32).view(np.float32)
    uvm[:, 3] = np.ones(n, np.uint32).view(np.float32)
    nrm = np.tile(np.array([0, 0, 1, 0], np.float32), (n, 1))
    pos = np.zeros((n, 4), np.float32)
    mat = np.tile(np.array([ax, ay, N, R], np.float32), (n, 1))
    return dict(duv=duv, uvm=uvm, nrm=nrm, pos=pos, mat=mat)


def _scene(wi, wo, ndf="ggx", seed=1):
    from paper_2306_05051_b200 import synth
    return synth.SceneParams(seed=seed, ndf=ndf, view_kind="directional", view=tuple(wi),
                             lights=[synth.Light("directional", tuple(wo), (1.0, 1.0, 1.0))])


def _dir(theta_deg, phi_deg):
    t, p = math.radians(theta_deg), math.radians(phi_deg)
    return (math.sin(t) * math.cos(p), math.sin(t) * math.sin(p), math.cos(t))


# ----------------------------------------------------------------------------- check 1
@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
@pytest.mark.parametrize("window,r_foot", [((12, 16), 1.0), ((6, 32), 5.333333)])
def test_check1_brute_force_facets(orc, ndf, window, r_foot):
    m = 32                      # N = 1024 stratified facets on the unit patch
    alpha, th_h, gamma = 0.5, math.radians(20.0), math.radians(12.0)
    h = np.array([math.sin(th_h), 0.0, math.cos(th_h)])
    # p_cone = int_cone D(m)(m.n) dw, by quadrature around h
    def integrand(t, p):
        a = np.array([math.sin(t) * math.cos(p), math.sin(t) * math.sin(p), math.cos(t)])
        # rotate cone axis from z to h
        c, s = math.cos(th_h), math.sin(th_h)
        mvec = np.array([c * a[0] + s * a[2], a[1], -s * a[0] + c * a[2]])
        return float(stats.ndf_D(ndf, alpha, alpha, mvec[None])[0]) * mvec[2] * math.sin(t)
    p_cone, _ = integrate.dblquad(lambda t, p: integrand(t, p), 0, 2 * math.pi, 0, gamma, epsabs=1e-8)
    rng = np.random.default_rng(11)
    M = 4000
    wx, wy = window
    area = wx * wy / (m * m)                       # 0.1875 in both layouts
    brute = np.empty(M, int)
    cosg = math.cos(gamma)
    for k in range(M):
        pts = stats.stratified_points(m, rng)
        nrm = stats.sample_ndf_normals(ndf, alpha, m * m, rng)
        inside = (pts[:, 0] < wx / m) & (pts[:, 1] < wy / m)
        in_cone = nrm @ h > cosg
        brute[k] = int((inside & in_cone).sum())
    # the distributed law through the oracle's lattice for a footprint of that
    # area and anisotropy: n_i = w_i N 2^ls_i, sum of exact binomials
    ls, lr, jo, w, _ = orc.lattice(area, r_foot, 0.0)
    n_i = [wi * m * m * 2.0 ** a for wi, a in zip(w, ls) if wi > 0]
    assert abs(sum(n_i) - 1024 * area) < 1e-3
    # fractional trial counts (reading R-4): Bin(floor n, p) + Bernoulli(frac(n) p),
    # the oracle's exact test sampler
    law = sum(rng.binomial(int(math.floor(x)), p_cone, M) + (rng.random(M) < (x - math.floor(x)) * p_cone)
              for x in n_i).astype(int)
    mean_ref = 1024 * area * p_cone
    assert abs(brute.mean() - mean_ref) < 4 * math.sqrt(mean_ref * (1 - p_cone) / M)
    assert abs(brute.var() / (mean_ref * (1 - p_cone)) - 1) < 0.1
    assert stats.chi2_two_sample(brute, law) > 1e-3


# ----------------------------------------------------------------------------- check 2
@pytest.mark.parametrize("sampler", ["exact", "gated"])
def test_check2_expected_count_is_NPp(orc, sampler):
    rng = np.random.default_rng(12)
    npx = 6
    uv = rng.random((npx, 2)).astype(np.float32) * 0.9
    # random anisotropic footprints of area ~2^-7.. with N chosen so N P ~ 30..200
    duv = []
    for i in range(npx):
        P = 2.0 ** rng.uniform(-9, -6)
        rr = 2.0 ** rng.uniform(0, 4)
        th = rng.uniform(0, math.pi)
        smax, smin = math.sqrt(P * rr), math.sqrt(P / rr)
        c, s = math.cos(th), math.sin(th)
        J = np.array([[c, -s], [s, c]]) @ np.diag([smax, smin])
        duv.append([J[0, 0], J[1, 0], J[0, 1], J[1, 1]])
    seeds = 300
    Cs = np.zeros((seeds, npx))
    ref = np.zeros(npx)
    for i in range(npx):
        g = _gbuf(duv[i], uv[i:i + 1], 2.0 ** rng.uniform(13, 14.5), 0.4, 0.4, 0.3)
        for sd in range(seeds):
            sc = _scene(_dir(30, 0), _dir(40, 140), seed=1000 + sd)
            _, _, rec = orc.eval(g, sc, debug=True, threads=1, sampler=sampler)
            r = rec[0, 0]
            Cs[sd, i] = r["C"]
            if sd == 0:
                if sampler == "exact":
                    ref[i] = float(np.sum(r["n"].astype(np.float64))) * float(r["p"])
                else:   # sum of the enumerated gated means of the 4 slots
                    ref[i] = sum(stats.pmf_mean(stats.gated_pmf_enumerated(float(x), float(r["p"]))[0])
                                 for x in r["n"] if x > 0)
    mean = Cs.mean(0)
    se = Cs.std(0, ddof=1) / math.sqrt(seeds)
    assert np.all(np.abs(mean - ref) < 4.5 * se + 1e-9), (mean, ref, se)


def test_check2_exact_sampler_variance(orc):
    """Var[b] = n p (1-p): with the exact sampler, a single-grid
    footprint on a lattice point (C1 layout, beta = (1,0,0)) has
    C = sum_j v_j b_j, so Var C = n p (1-p) sum_j v_j^2."""
    g = _gbuf([1 / 64, 0, 0, 1 / 64], np.array([[10 / 64, 20 / 64]], np.float32), 1e5 * 4, 0.3, 0.3, 0.2)
    Cs = []
    for sd in range(3000):
        _, _, rec = orc.eval(g, _scene(_dir(30, 0), _dir(30, 180), seed=sd), debug=True, threads=1,
                             sampler="exact")
        Cs.append(rec[0, 0]["C"])
    r = rec[0, 0]
    n, p = float(r["n"][0]), float(r["p"])
    assert n == 97.65625 and abs(p - 0.2) < 1e-6
    var_ref = n * p * (1 - p) * 4 * (0.25 ** 2)      # v_j = 1/4 (h = n -> g = -1/2)
    assert abs(np.var(Cs) / var_ref - 1) < 0.1


# ----------------------------------------------------------------------------- check 3
@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
def test_check3_convergence_to_smooth_ndf(orc, ndf):
    """Mean over spatial offsets of D_P(h) -> D(h) as the number of facets per
    footprint N P grows: the per-pixel spread shrinks monotonically wherever
    the expected count N P p is >= 1, and the mean is within 2 % from N P = 1e6
    (S:L409 'density 10^6 facets/footprint')."""
    rng = np.random.default_rng(13)
    uv = rng.random((2048, 2)).astype(np.float32)
    alpha = 0.35
    for th_h in (0.0, 10.0, 20.0, 30.0, 45.0):
        wi = _dir(th_h + 5.0, 0.0)
        wo = _dir(max(th_h - 5.0, 0.0) if th_h >= 5 else 5.0 - th_h, 0.0 if th_h >= 5 else 180.0)
        hv = np.array(wi) + np.array(wo)
        hv /= np.linalg.norm(hv)
        D_h = float(stats.ndf_D(ndf, alpha, alpha, hv[None])[0])
        spreads, means, counts = [], [], []
        for NP in (1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8):
            g = _gbuf([1 / 8, 0, 0, 1 / 8], uv, NP * 64, alpha, alpha, 0.2)
            _, _, rec = orc.eval(g, _scene(wi, wo, ndf), debug=True)
            Dp = rec[:, 0]["Dp"].astype(np.float64)
            means.append(Dp.mean() / D_h - 1)
            spreads.append(np.sqrt(np.mean((Dp / D_h - 1) ** 2)))
            counts.append(NP * float(rec[0, 0]["p"]))
        for i in range(len(spreads) - 1):
            if counts[i] >= 1.0:
                assert spreads[i + 1] < spreads[i], (th_h, spreads, counts)
        assert all(abs(m) < 0.02 for m in means[4:]), (th_h, means)


# ----------------------------------------------------------------------------- check 4
def test_check4_lod_coherence(orc):
    """Sweep the footprint area over [2^(k-1), 2^(k+1)] at fixed surface points:
    (a) level-k texels keep the same seeds (hashes) over the whole sweep (the
    seeds depend only on lattice indices, reading R-24); (b) at P = 2^k the left
    and right limits of the blended count agree almost surely."""
    rng = np.random.default_rng(14)
    k = -10
    uv = rng.random((64, 2)).astype(np.float32)
    sc = _scene(_dir(20, 0), _dir(25, 160))
    Ps = np.float32(2.0 ** np.linspace(k - 1, k + 1, 81)[1:-1])
    level_hashes = [dict() for _ in range(len(uv))]
    for P in Ps:
        s = math.sqrt(float(P))
        g = _gbuf([s, 0, 0, s], uv, 2.0 ** 16, 0.3, 0.3, 0.5)
        _, _, rec = orc.eval(g, sc, debug=True)
        for i, r in enumerate(rec[:, 0]):
            for slot in range(4):
                if r["ls"][slot] == k and r["w"][slot] > 0:
                    hs = tuple(r["hash"][slot * 12:(slot + 1) * 12])
                    level_hashes[i].setdefault(hs, 0)
                    level_hashes[i][hs] += 1
    assert all(len(d) == 1 for d in level_hashes)
    # (b) left/right limits at the LOD boundary P = 2^k
    diffs = 0
    total = 0
    uv2 = rng.random((4000, 2)).astype(np.float32)
    left = math.sqrt(float(np.nextafter(np.float32(2.0 ** k), np.float32(0))))
    gl = _gbuf([left, 0, 0, left], uv2, 2.0 ** 16, 0.3, 0.3, 0.5)
    gr = _gbuf([math.sqrt(2.0 ** k), 0, 0, math.sqrt(2.0 ** k)], uv2, 2.0 ** 16, 0.3, 0.3, 0.5)
    _, _, rl = orc.eval(gl, sc, debug=True)
    _, _, rr = orc.eval(gr, sc, debug=True)
    Cl, Cr = rl[:, 0]["C"], rr[:, 0]["C"]
    assert rl[0, 0]["P"] < 2.0 ** k <= rr[0, 0]["P"]
    assert np.mean(np.abs(Cl - Cr) > 1e-3 * np.maximum(Cl, 1.0)) < 0.02
