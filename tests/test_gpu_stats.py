"""GPU statistics harness: the device draw function, driven
at scale through the C ABI (debug records), against the laws the oracle
enumerates -- Fig. 9 (gated approximation vs its law over an (n, p) grid,
P:L933-972), Fig. 4 (distributing vs blending LODs, Eq. 7 vs
Eq. 10) and the expectation check (north-star check 2) with 10^5-10^6 draws."""
import math

import numpy as np
import pytest
import torch

from oracle import stats

pytestmark = pytest.mark.gpu

S30, C30 = math.sin(math.radians(30)), math.cos(math.radians(30))


@pytest.fixture(scope="module")
def ctx():
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import build
    build.build()
    c = pkg.Context(0)
    yield c
    c.close()


def _gbuffer(M, P, N, R, alpha=0.3, seed=0, aniso=None):
    """M pixels with the same footprint of area P (isotropic unless aniso=(r,
    psi)), distinct object ids (independent seeds) and random uv."""
    from paper_2306_05051_b200 import synth
    g = torch.Generator().manual_seed(seed)
    H, W = M // 256, 256
    duv = torch.zeros(H, W, 4)
    if aniso is None:
        s = math.sqrt(P)
        duv[..., 0] = s
        duv[..., 3] = s
    else:
        r, th = aniso
        smax, smin = math.sqrt(P * r), math.sqrt(P / r)
        c, sn = math.cos(th), math.sin(th)
        duv[..., 0], duv[..., 1] = c * smax, sn * smax
        duv[..., 2], duv[..., 3] = -sn * smin, c * smin
    uvm = torch.zeros(H, W, 4)
    uvm[..., :2] = torch.rand(H, W, 2, generator=g)
    obj = torch.arange(H * W, dtype=torch.int64).reshape(H, W) * 2654435761 + seed * 97
    uvm[..., 2] = synth._bits_to_f32(obj)
    uvm[..., 3] = synth._bits_to_f32(torch.ones(H, W, dtype=torch.int64))
    nrm = torch.zeros(H, W, 4)
    nrm[..., 2] = 1.0
    mat = torch.tensor([alpha, alpha, N, R]).expand(H, W, 4).contiguous()
    return synth.GBuffer(duv.contiguous(), uvm.contiguous(), nrm.contiguous(), torch.zeros(H, W, 4), mat)


def _mirror_scene(seed=1):
    from paper_2306_05051_b200 import synth
    return synth.SceneParams(seed=seed, ndf="ggx", view_kind="directional", view=(S30, 0.0, C30),
                             lights=[synth.Light("directional", (-S30, 0.0, C30), (1.0, 1.0, 1.0))])


def _records(ctx, gb, sc):
    import paper_2306_05051_b200 as pkg
    out, rec = pkg.glint_eval(ctx, gb.to("cuda"), sc, debug=True)
    torch.cuda.synchronize()
    return out, rec[:, 0]


@pytest.mark.parametrize("n,R", [(1.0, 0.05), (4.0, 0.3), (16.0, 0.5), (64.0, 0.95), (24.4140625, 0.034),
                                 (400.0, 0.2)])
def test_fig9_device_draws_follow_the_gated_law(ctx, n, R):
    """Single grid of n trials (P = 2^-12, N = n 2^12), p = R (h = n): the
    12 draws of 2^17 pixels (1.5e6 draws) follow the contract's exact law
    (chi-square); the distance to the exact binomial is reported."""
    M = 1 << 17
    gb = _gbuffer(M, 2.0 ** -12, n * 4096.0, R)
    out, r = _records(ctx, gb, _mirror_scene())
    assert np.all(r["n"][:, 0] == np.float32(n)) and np.all(r["n"][:, 1:] == 0)
    p = float(r["p"][0])
    assert abs(p - R) < 1e-6 * R + 1e-9
    c = r["count"][:, :12].ravel().astype(np.int64)
    pmf, (T, *_x) = stats.gated_pmf_enumerated(float(np.float32(n)), p)
    assert np.all(r["T"][:, 0] == T)
    pv = stats.chi2_gof(np.bincount(c, minlength=len(pmf)), pmf)
    assert pv > 1e-4, (n, R, pv)
    if n == int(n):
        tv = stats.total_variation(np.bincount(c, minlength=len(pmf)) / len(c), stats.binom_pmf(int(n), p))
        print(f"n={n} p={p}: TV(device draws, exact binomial) = {tv:.3f}")


def test_fig4_distributing_vs_blending_on_device(ctx):
    """N = 64, p = 1/2, footprint 0.375 between the LOD areas 0.25 and 0.5:
    the device's distributed draw b(8) + b(16) (two grids, same draw index)
    follows the convolution of the two gated laws, mean 12 and variance ~6 as
    Binomial(24, 1/2); Zirr's output mix of the full-LOD draws (Eq. 7) has the
    same mean but about half the variance (Fig. 4 b vs c)."""
    M = 1 << 16
    sc = _mirror_scene()
    R = 0.5
    _, r = _records(ctx, _gbuffer(M, 0.375, 64.0, R, seed=3), sc)
    n = r["n"][0]
    assert sorted(np.round(n[n > 0], 4).tolist()) == [8.0, 16.0]
    slots = [int(i) for i in np.nonzero(n > 0)[0]]
    p = float(r["p"][0])
    dist = (r["count"][:, slots[0] * 12:(slots[0] + 1) * 12] + r["count"][:, slots[1] * 12:(slots[1] + 1) * 12])
    dist = dist.ravel().astype(np.int64)
    law = np.convolve(stats.gated_pmf_enumerated(float(n[slots[0]]), p)[0],
                      stats.gated_pmf_enumerated(float(n[slots[1]]), p)[0])
    assert stats.chi2_gof(np.bincount(dist, minlength=len(law)), law) > 1e-4
    assert abs(dist.mean() - 12.0) < 0.6 and abs(dist.var() / 6.0 - 1) < 0.15
    # Zirr: blend full-weight draws of the two LODs (footprints exactly 0.5 and 0.25)
    _, r_hi = _records(ctx, _gbuffer(M, 0.5, 64.0, R, seed=3), sc)
    _, r_lo = _records(ctx, _gbuffer(M, 0.25, 64.0, R, seed=3), sc)
    # sqrt(0.5)^2 rounds just below 0.5 in fp32: take the dominant grid
    ih, il = int(np.argmax(r_hi["n"][0])), int(np.argmax(r_lo["n"][0]))
    assert abs(r_hi["n"][0, ih] - 32.0) < 1e-4 and abs(r_lo["n"][0, il] - 16.0) < 1e-4
    c_hi = r_hi["count"][:, ih * 12:(ih + 1) * 12].ravel()
    c_lo = r_lo["count"][:, il * 12:(il + 1) * 12].ravel()
    zirr = 0.5 * c_hi + 0.5 * c_lo
    assert abs(zirr.mean() - dist.mean()) < 0.8
    assert zirr.var() < 0.65 * dist.var()


def test_expectation_at_scale(ctx):
    """North-star check 2 on the device: over 2^18 pixels with a random
    anisotropic footprint the mean of each grid's count equals the contract's
    enumerated gated mean E(n_i, p), so E[C] = sum_i E(n_i, p) (and -> N P p as
    N P p grows)."""
    M = 1 << 18
    gb = _gbuffer(M, 2.0 ** -9.3, 2.0 ** 15, 0.2, aniso=(5.7, 0.7), seed=5)
    _, r = _records(ctx, gb, _mirror_scene())
    p = float(r["p"][0])
    for i in range(4):
        ni = float(r["n"][0, i])
        if ni <= 0:
            continue
        c = r["count"][:, i * 12:(i + 1) * 12].ravel().astype(np.float64)
        pmf, _ = stats.gated_pmf_enumerated(ni, p)
        m = stats.pmf_mean(pmf)
        se = math.sqrt(float(np.dot((np.arange(len(pmf)) - m) ** 2, pmf)) / len(c)) * 2.0  # draws share seeds
        assert abs(c.mean() - m) < 4 * se + 1e-12, (i, ni, c.mean(), m, se)


def test_convergence_to_smooth_ndf_on_device(ctx):
    """North-star check 3 on the device (Eq. 5-6): over 256^2 independent
    surface points, D_P / D(h) has mean -> 1 and a spread that shrinks about
    sqrt(10)-fold per decade of N P (tools/gpu/convergence.py at full scale)."""
    import importlib.util
    import os
    import paper_2306_05051_b200 as pkg
    from paper_2306_05051_b200 import synth
    spec = importlib.util.spec_from_file_location(
        "convergence", os.path.join(os.path.dirname(__file__), "..", "tools", "gpu", "convergence.py"))
    cv = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(cv)
    dev = torch.device("cuda", 0)
    n, P = 256, 2.0 ** -10
    t, e = math.radians(20.0), math.radians(5.0)
    sc = synth.SceneParams(seed=3, ndf="ggx", view_kind="directional", view=(math.sin(t + e), 0.0, math.cos(t + e)),
                           lights=[synth.Light("directional", (math.sin(t - e), 0.0, math.cos(t - e)), (1.0, 1.0, 1.0))])
    ref = pkg.glint_eval(ctx, cv.quad(n, P, 2.0 ** 40, 0.35, dev), sc)[..., 0].double().mean().item()
    spreads = []
    for NP in (1e3, 1e4, 1e5, 1e6):
        L = pkg.glint_eval(ctx, cv.quad(n, P, NP / P, 0.35, dev), sc)[..., 0].double() / ref
        spreads.append(float(L.std()))
        if NP >= 1e5:
            assert abs(float(L.mean()) - 1) < 0.01
    for a, b in zip(spreads, spreads[1:]):
        assert 2.3 < a / b < 4.3, spreads
