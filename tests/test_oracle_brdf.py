"""Pins for the NDF ratio (Eq. 4; targets P:L148, L1211), the BRDF
shell (Eq. 1-2; readings R-21, R-22) against quadrature, textbook
closed forms and reciprocity."""
import math

import numpy as np
import pytest
from scipy import integrate

from oracle import stats


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
@pytest.mark.parametrize("ax,ay", [(0.3, 0.3), (1.0, 1.0), (0.2, 0.5)])
def test_ndf_projected_area_normalisation(orc, ndf, ax, ay):
    """int D(h) cos(theta_h) dw = 1 with D = D(n) * ratio(h), D(n) = 1/(pi ax ay)."""
    Dn = 1.0 / (math.pi * ax * ay)

    def f(th, ph):
        h = (math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th))
        return Dn * orc.ratio(ndf, ax, ay, *h) * math.cos(th) * math.sin(th)

    val, _ = integrate.dblquad(lambda th, ph: f(th, ph), 0, 2 * math.pi, 0, math.pi / 2,
                               epsabs=1e-5, epsrel=1e-5)
    assert abs(val - 1.0) < 5e-3, val


def test_ratio_closed_forms(orc):
    assert abs(orc.ratio("ggx", 0.3, 0.3, 0.0, 0.0, 1.0) - 1.0) < 1e-6      # h = n -> 1
    assert abs(orc.ratio("beckmann", 0.3, 0.3, 0.0, 0.0, 1.0) - 1.0) < 1e-6
    s = math.sqrt(0.5)                                                         # Beckmann a=1, 45 deg: 4/e
    assert abs(orc.ratio("beckmann", 1.0, 1.0, s, 0.0, s) - 4 / math.e) < 2e-6
    h = np.array([0.3, -0.2, math.sqrt(1 - 0.13)])
    for ndf in ("ggx", "beckmann"):
        ref = stats.ndf_D(ndf, 0.25, 0.4, h) * math.pi * 0.25 * 0.4
        assert abs(orc.ratio(ndf, 0.25, 0.4, *h) - ref) < 2e-6 * max(1, ref)
    assert orc.ratio("ggx", 0.3, 0.3, 1.0, 0.0, 0.0) == 0.0                    # grazing h


def test_schlick():
    import oracle
    assert abs(oracle.schlick(0.04, 0.5) - 0.07) < 1e-15
    assert oracle.schlick(0.3, 1.0) == 0.3 and oracle.schlick(0.3, 0.0) == 1.0


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
def test_smith_g1_vs_exact_lambda(orc, ndf):
    """With wo = n (Lambda = 0), G2 = G1(wi) = 1/(1 + Lambda(wi)); GGX exact,
    Beckmann's rational fit within 0.5 % of the erf form."""
    for alpha in (0.1, 0.3, 0.7, 1.0):
        for th in np.linspace(0.05, 1.5, 20):
            wi = (math.sin(th), 0.0, math.cos(th))
            g = orc.smith_g2(ndf, alpha, alpha, wi, (0.0, 0.0, 1.0))
            ref = 1.0 / (1.0 + stats.smith_lambda_exact(ndf, alpha, math.cos(th)))
            assert abs(g - ref) < (1e-12 if ndf == "ggx" else 5e-3 * ref)


def test_negative_zero_normal_frames_agree(orc):
    """n_z = -0 (a normal in the tangent plane): the fp32 decision frame and
    the fp64 radiance frame take the same branch of the Duff et al. ONB
    (sgn = copysign(1, n_z) = -1), so anisotropic G2 matches its fp64 value
    computed with that frame."""
    import math
    from paper_2306_05051_b200 import synth
    g = dict(duv=np.array([[0.01, 0, 0, 0.01]], np.float32),
             uvm=np.concatenate([np.array([[0.3, 0.4]], np.float32), np.array([[5]], np.uint32).view(np.float32),
                                 np.array([[1]], np.uint32).view(np.float32)], 1),
             nrm=np.array([[0.9, -0.3, -0.0, 0]], np.float32), pos=np.zeros((1, 4), np.float32),
             mat=np.array([[0.2, 0.7, 1e7, 0.3]], np.float32))
    sc_n = synth.SceneParams(seed=2, view_kind="directional", view=(0.6, 0.5, 0.3),
                             lights=[synth.Light("directional", (0.7, -0.1, 0.4), (1, 1, 1))])
    r_neg = orc.eval(g, sc_n)[0]
    g["nrm"][0, 2] = np.float32(-1e-30)       # same frame branch (negative), same geometry to fp32
    r_tiny = orc.eval(g, sc_n)[0]
    assert r_neg[0, 0] > 0 and abs(r_neg[0, 0] / r_tiny[0, 0] - 1) < 1e-5


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
@pytest.mark.parametrize("alpha", [0.1, 0.35, 0.8])
def test_white_furnace_of_the_smooth_model(orc, ndf, alpha):
    """with F = 1, the smooth microfacet BRDF the glints
    converge to (D from the oracle's ratio, the oracle's height-correlated G2)
    reflects at most 1 + 2 % of the incoming energy:
    int D(h) G2(wi, wo) / (4 n.wi) dwo <= 1.02. (Single scattering loses energy:
    at normal incidence the part of the NDF beyond theta_h = 45 deg reflects
    below the horizon, 1 - 1/(alpha^2 + 1) of it for GGX.)"""
    Dn = 1.0 / (math.pi * alpha * alpha)
    for th_i in (0.0, 0.5, 1.0, 1.3):
        wi = np.array([math.sin(th_i), 0.0, math.cos(th_i)])
        n_t, n_p = 160, 240
        ths = (np.arange(n_t) + 0.5) * (math.pi / 2) / n_t
        phs = (np.arange(n_p) + 0.5) * 2 * math.pi / n_p
        total = 0.0
        for th in ths:
            for ph in phs:
                wo = np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
                h = wi + wo
                h /= np.linalg.norm(h)
                D = Dn * orc.ratio(ndf, alpha, alpha, *h)
                G2 = orc.smith_g2(ndf, alpha, alpha, wi, wo)
                total += D * G2 / (4 * wi[2]) * math.sin(th)
        total *= (math.pi / 2 / n_t) * (2 * math.pi / n_p)
        assert total <= 1.02, (ndf, alpha, th_i, total)
        if th_i == 0.0 and ndf == "ggx" and alpha <= 0.35:   # G2 ~ 1: the projected NDF mass within 45 deg
            assert 0.9 / (alpha * alpha + 1) < total <= 1.0 / (alpha * alpha + 1) + 5e-3, (alpha, total)
        if alpha <= 0.35 and th_i <= 1.0:
            assert total > 0.75, (ndf, alpha, th_i, total)
