"""Pins for the light and view branches of the oracle (S5 decisions, S9 shell):
point lights and pinhole views against directional ones and against a
hand-computed case, the multi-light sum, and the reciprocity of the radiance
shell (Eq. 1-2; punctual lights P:L1228, reading R-27: point
E = I / d^2, w_i = normalize(view - pos), w_o = normalize(light - pos)).

Exactness trick: positions on a dyadic grid and lights / cameras at small
integer offsets from them, so light - pos and view - pos are exact in fp32. A
point light then takes the fp32 decision path of the directional light whose
(unnormalised) direction is that difference, bit for bit, and only the
irradiance differs: E = I / |d|^2 exactly. A sign slip (pos - light) or a
wrong falloff fails these by orders of magnitude."""
import math

import numpy as np
import pytest

from paper_2306_05051_b200 import synth


def _dyadic_gbuffer(h, w, seed):
    """random_gbuffer with positions on the 1/8 grid in [-2, 2]^2 x [0, 1/2]
    (so light - pos is exact in fp32 for the integer light offsets below)."""
    gb = synth.random_gbuffer(h, w, seed=seed)
    rng = np.random.default_rng(seed)
    pos = gb.pos.clone()
    pos[..., 0] = torch_from(rng.integers(-16, 17, (h, w)) / 8.0)
    pos[..., 1] = torch_from(rng.integers(-16, 17, (h, w)) / 8.0)
    pos[..., 2] = torch_from(rng.integers(0, 5, (h, w)) / 8.0)
    return synth.GBuffer(gb.duv, gb.uvm, gb.nrm, pos, gb.mat)


def torch_from(a):
    import torch
    return torch.as_tensor(np.asarray(a, np.float32))


def _pixel_frames(gb):
    """Split a G-buffer into 1-pixel buffers (each gets its own scene)."""
    planes = [p.reshape(-1, 4) for p in gb.planes()]
    for i in range(planes[0].shape[0]):
        yield i, synth.GBuffer(*[p[i:i + 1].reshape(1, 1, 4) for p in planes])


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
def test_point_light_equals_directional_times_inverse_square(orc, ndf):
    """A point light at L and, pixel by pixel, a directional light along the
    exact fp32 difference d = L - pos: identical records (hashes, counts, p,
    nodes) and rgb_point = rgb_dir / |d|^2 (I / d^2 falloff) to fp64 rounding."""
    gb = _dyadic_gbuffer(6, 7, seed=21)
    L = (3.0, -2.0, 6.0)
    view = synth.SceneParams(seed=5, ndf=ndf, beta=0.03, f0=(0.04, 0.5, 0.95),
                             view_kind="directional", view=(0.2, -0.3, 0.9))
    nz = 0
    for i, g1 in _pixel_frames(gb):
        p = g1.pos.reshape(4).numpy().astype(np.float64)
        d = tuple(float(L[k] - p[k]) for k in range(3))
        assert all(np.float32(L[k]) - np.float32(p[k]) == np.float32(d[k]) for k in range(3))
        sc_p = synth.SceneParams(**{**view.__dict__, "lights": [synth.Light("point", L, (7.0, 11.0, 13.0))]})
        sc_d = synth.SceneParams(**{**view.__dict__, "lights": [synth.Light("directional", d, (7.0, 11.0, 13.0))]})
        rp, fp, recp = orc.eval(g1, sc_p, debug=True)
        rd, fd, recd = orc.eval(g1, sc_d, debug=True)
        assert np.array_equal(fp, fd)
        for f in ("hash", "count", "p", "cx0", "cy0", "T", "light_active"):
            assert np.array_equal(recp[f], recd[f]), (i, f)
        d2 = sum(x * x for x in d)
        np.testing.assert_allclose(rp, rd / d2, rtol=1e-13, atol=0)
        nz += int(rp[0, 0] > 0)
    assert nz >= 5           # the comparison saw glints


def test_pinhole_view_equals_directional_view(orc):
    """A pinhole camera at c and, pixel by pixel, a directional view along the
    exact difference c - pos: bit-identical records and radiance."""
    gb = _dyadic_gbuffer(6, 7, seed=22)
    cam = (-1.0, -3.0, 5.0)
    lights = [synth.Light("point", (2.0, 1.0, 4.0), (5.0, 5.0, 5.0)),
              synth.Light("directional", (0.1, 0.4, 0.8), (1.0, 2.0, 3.0))]
    nz = 0
    for i, g1 in _pixel_frames(gb):
        p = g1.pos.reshape(4).numpy().astype(np.float64)
        v = tuple(float(cam[k] - p[k]) for k in range(3))
        sc_c = synth.SceneParams(seed=9, beta=0.04, view_kind="point", view=cam, lights=lights)
        sc_v = synth.SceneParams(seed=9, beta=0.04, view_kind="directional", view=v, lights=lights)
        rc, fc, recc = orc.eval(g1, sc_c, debug=True)
        rv, fv, recv = orc.eval(g1, sc_v, debug=True)
        assert np.array_equal(fc, fv) and np.array_equal(recc.view(np.uint8), recv.view(np.uint8)), i
        assert np.array_equal(rc, rv), i
        nz += int(rc[0, 0] > 0)
    assert nz >= 5


def test_reversed_light_is_below_the_horizon(orc):
    """The sign of d = light - pos: a point light below the surface point (or a
    directional light pointing into the surface) contributes nothing."""
    g = synth.c1("ggx", "mirror")
    s30, c30 = math.sin(math.radians(30)), math.cos(math.radians(30))
    up = synth.SceneParams(seed=1, view_kind="directional", view=(s30, 0.0, c30),
                           lights=[synth.Light("point", (0.5 - 5 * s30, 0.5, 5 * c30), (25.0, 25.0, 25.0))])
    down = synth.SceneParams(**{**up.__dict__, "lights": [synth.Light("point", (0.5 - 5 * s30, 0.5, -5 * c30),
                                                                       (25.0, 25.0, 25.0))]})
    assert orc.eval(g.gbuf, up)[0].max() > 0
    r, _, rec = orc.eval(g.gbuf, down, debug=True)
    assert r.max() == 0 and rec["light_active"].max() == 0


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
def test_pinhole_point_light_mirror_hand_computed(orc, ndf):
    """C1's quad (n = +z) seen by a pinhole camera at distance 10 along the
    30-degree view direction from pixel (32, 32), lit by a point light at
    distance 10 along the mirror direction (I = 100, so E = 1): h = n, so
    p = R (ratio 1, Eq. 4), and the pixel's radiance is, by hand,
    F(cos 30) G2 C / (pi a^2 R N P) / (4 cos 30) with Schlick F, the GGX /
    Beckmann-Walter Smith G2 at 30 degrees on both sides, and the blended count
    C from the record."""
    import torch
    fr = synth.c1(ndf, "mirror")
    i = 32 * 64 + 32
    g1 = synth.GBuffer(*[p.reshape(-1, 4)[i:i + 1].reshape(1, 1, 4) for p in fr.gbuf.planes()])
    x0 = g1.pos.reshape(4)[:3].double().numpy()
    s30, c30 = 0.5, math.sqrt(3) / 2
    cam = tuple(float(np.float32(x0[k] + 10 * (s30, 0.0, c30)[k])) for k in range(3))
    lit = tuple(float(np.float32(x0[k] + 10 * (-s30, 0.0, c30)[k])) for k in range(3))
    f0 = 0.3
    sc = synth.SceneParams(seed=3, ndf=ndf, f0=(f0, f0, f0), view_kind="point", view=cam,
                           lights=[synth.Light("point", lit, (100.0, 100.0, 100.0))])
    best = None
    for seed in range(1, 200):          # a seed where this pixel glints
        sc.seed = seed
        rgb, fl, rec = orc.eval(g1, sc, debug=True)
        if rec["C"][0, 0] > 0:
            best = (rgb, rec)
            break
    assert best is not None
    rgb, rec = best
    assert abs(rec["p"][0, 0] / np.float32(0.034) - 1) < 1e-6           # h = n -> p = R
    a, R, N, P = 0.3, np.float32(0.034), np.float32(1e5), 2.0 ** -12
    F = f0 + (1 - f0) * (1 - c30) ** 5
    if ndf == "ggx":
        lam = 0.5 * (-1 + math.sqrt(1 + a * a * (1 - c30 * c30) / (c30 * c30)))
    else:
        t = c30 / (a * math.sqrt(1 - c30 * c30))
        lam = 0.0 if t >= 1.6 else (1 - 1.259 * t + 0.396 * t * t) / (3.535 * t + 2.181 * t * t)
    G2 = 1 / (1 + 2 * lam)
    d = np.array(lit) - x0
    E = 100.0 / float(d @ d)
    ref = F * G2 * float(rec["C"][0, 0]) / (math.pi * a * a * float(R) * float(N) * P) * E / (4 * c30)
    np.testing.assert_allclose(rgb[0], ref, rtol=2e-6)   # camera/light rounded to fp32, C an fp32 record


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
def test_multi_light_is_the_sum_of_single_light_renders(orc, ndf):
    """L lights (point and directional) = the sum of L one-light renders:
    each light's records equal its one-light render's bit for bit, radiance
    sums to fp64 rounding, flags are the OR."""
    gb = synth.random_gbuffer(9, 11, seed=31)
    sc = synth.random_scene(31, n_lights=5, ndf=ndf)
    rgb, fl, rec = orc.eval(gb, sc, debug=True)
    tot = np.zeros_like(rgb)
    flo = np.zeros_like(fl)
    for l, lt in enumerate(sc.lights):
        s1 = synth.SceneParams(**{**sc.__dict__, "lights": [lt]})
        r1, f1, rec1 = orc.eval(gb, s1, debug=True)
        tot += r1
        flo |= f1
        keep = [n for n in rec.dtype.names if n not in ("flags",)]
        for n in keep:
            assert np.array_equal(rec[n][:, l], rec1[n][:, 0]), (l, n)
    assert np.array_equal(fl, flo)
    assert rgb.max() > 0
    np.testing.assert_allclose(rgb, tot, rtol=1e-13, atol=0)


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
def test_radiance_shell_reciprocity(orc, ndf):
    """Eq. 1-2: the BRDF f = F G2 D_P / (4 (n.wi)(n.wo)) is symmetric in
    (wi, wo), so the shell's contribution L = f E (n.wo) times (n.wi) is: at a
    fixed D_P, swapping a directional view and a directional light leaves
    L (n.wi) unchanged to fp64 rounding (a swapped F or G term, or the wrong
    cosine in the denominator, breaks it at O(1))."""
    rng = np.random.default_rng(8)
    for _ in range(40):
        n = rng.standard_normal(3)
        n[2] = abs(n[2]) + 0.1
        n = n.astype(np.float32)
        a = rng.standard_normal(3).astype(np.float32)
        b = rng.standard_normal(3).astype(np.float32)
        ax, ay = [float(np.float32(x)) for x in 0.05 + 0.8 * rng.random(2)]
        f0 = tuple(float(np.float32(x)) for x in rng.random(3))

        def shell(view, light):
            sc = synth.SceneParams(ndf=ndf, f0=f0, view_kind="directional", view=tuple(map(float, view)),
                                   lights=[synth.Light("directional", tuple(map(float, light)), (1.0, 1.0, 1.0))])
            return orc.shell(sc, 0, n, (0.0, 0.0, 0.0), ax, ay, 0.37)

        (r1, ok1), (r2, ok2) = shell(a, b), shell(b, a)
        nn = n.astype(float) / np.linalg.norm(n.astype(float))
        ca = float(nn @ (a / np.linalg.norm(a.astype(float))))
        cb = float(nn @ (b / np.linalg.norm(b.astype(float))))
        assert ok1 == ok2 == (ca > 0 and cb > 0)
        if ok1:
            np.testing.assert_allclose(r1 * ca, r2 * cb, rtol=1e-12, atol=0)


def test_shell_zero_when_nothing_reflects_or_below_horizon(orc):
    """D_P = 0 adds exactly nothing (no 0 * inf), and so does an fp64 cosine
    <= 0, even with an overflowing irradiance."""
    sc = synth.SceneParams(view_kind="directional", view=(0.0, 0.3, 1.0),
                           lights=[synth.Light("point", (0.0, 0.0, 1e-19), (3e38, 3e38, 3e38))])
    r, ok = orc.shell(sc, 0, (0, 0, 1), (0, 0, 0), 0.3, 0.3, 0.0)
    assert not ok and np.all(r == 0)
    r, ok = orc.shell(sc, 0, (0, 0, 1), (0, 0, 0), 0.3, 0.3, 1.0)
    assert ok and np.all(np.isfinite(r)) and r[0] > 1e70         # fp64 holds I / d^2 = 3e76
    sc.view = (0.0, 1.0, -1e-9)                                   # view below the horizon
    r, ok = orc.shell(sc, 0, (0, 0, 1), (0, 0, 0), 0.3, 0.3, 1.0)
    assert not ok and np.all(r == 0)


@pytest.mark.parametrize("ndf", ["ggx", "beckmann"])
def test_whole_eval_reciprocity_tight(orc, ndf):
    """Swapping view and light over the whole pixel path: every count is
    identical (h is symmetric to fp32 rounding and no count flips here), and
    rgb (n.wi) is symmetric within the angular weights' sensitivity to that
    rounding, |dv/dh| ~ 1 / beta: with beta = 4 this is below 1e-6."""
    rng = np.random.default_rng(7)
    checked = 0
    for _ in range(16):
        a = rng.standard_normal(3); a[2] = abs(a[2]) + 0.2; a /= np.linalg.norm(a)
        b = rng.standard_normal(3); b[2] = abs(b[2]) + 0.2; b /= np.linalg.norm(b)
        a, b = a.astype(np.float32).astype(float), b.astype(np.float32).astype(float)
        fr = synth.c1(ndf, "mirror")
        fr.scene.beta = 4.0
        fr.scene.lights[0] = synth.Light("directional", tuple(b), (1.0, 1.0, 1.0))
        fr.scene.view = tuple(a)
        rgb1, _, rec1 = orc.eval(fr.gbuf, fr.scene, debug=True)
        fr.scene.lights[0] = synth.Light("directional", tuple(a), (1.0, 1.0, 1.0))
        fr.scene.view = tuple(b)
        rgb2, _, rec2 = orc.eval(fr.gbuf, fr.scene, debug=True)
        if not np.array_equal(rec1["count"], rec2["count"]):
            continue       # a count flipped on a 1-ulp difference of h: no symmetry to test
        na, nb = a[2] / np.linalg.norm(a), b[2] / np.linalg.norm(b)
        checked += int(rgb1.max() > 0)
        np.testing.assert_allclose(rgb1 * na, rgb2 * nb, rtol=1e-6, atol=0)
    assert checked >= 4
