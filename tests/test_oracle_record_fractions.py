"""Pins for the debug record's fraction fields (glint.h 2.1): the simplex cell
fractions of S3 (the barycentrics' arguments), the angular cell
fractions of Eq. 14 (v_j's arguments) and P>=1 of Eq. 16
(P:L989-996), each against something other than the record itself:

* sfx, sfy against the lattice vertices the same record holds (the triangle
  they pick, R-15) and against the grid coordinates recomputed through the
  exported grid transform (floor + fraction reassembles the coordinate);
* afx, afy against the half vector computed in fp64 from a hand-set
  directional view and light over a flat normal: cx0 + afx = h_x / beta - 1/2;
* pge1 against the closed form 1 - (1 - p)^n in fp64 and against the gate
  threshold T = ceil(P>=1 2^23) of the same record."""
import math

import numpy as np
import pytest

from paper_2306_05051_b200 import synth


def _records(orc, gb, sc):
    _, _, rec = orc.eval(gb, sc, debug=True)
    return rec


def test_simplex_fractions_pick_the_recorded_triangle(orc):
    gb = synth.random_gbuffer(12, 17, seed=31)
    sc = synth.random_scene(31, n_lights=2)
    rec = _records(orc, gb, sc)
    uvm = gb.uvm.reshape(-1, 4).numpy()
    checked = 0
    for px in range(rec.shape[0]):
        r = rec[px, 0]
        if not rec[px, :]["light_active"].any():
            continue
        for i in range(4):
            if not (r["w"][i] > 0):
                continue
            fx, fy = r["sfx"][i], r["sfy"][i]
            assert 0.0 <= fx < 1.0 and 0.0 <= fy < 1.0
            x0, y0 = int(r["lx"][3 * i]), int(r["ly"][3 * i])
            v1 = (int(r["lx"][3 * i + 1]), int(r["ly"][3 * i + 1]))
            v2 = (int(r["lx"][3 * i + 2]), int(r["ly"][3 * i + 2]))
            wrap = lambda a: (a + 2**31) % 2**32 - 2**31   # the record keeps the low 32 bits
            assert v1 == ((wrap(x0 + 1), y0) if fx >= fy else (x0, wrap(y0 + 1)))
            assert v2 == (wrap(x0 + 1), wrap(y0 + 1))
            # the grid coordinates through the exported transform: floor + fraction
            x, y = orc.grid_uv(float(uvm[px, 0]), float(uvm[px, 1]), int(r["ls"][i]), int(r["lr"][i]), int(r["jo"][i]))
            xs = np.float32(np.float32(x) + np.float32(0.5) * np.float32(y))
            assert np.float32(xs - np.floor(xs)) == fx
            assert np.float32(np.float32(y) - np.floor(np.float32(y))) == fy
            assert wrap(int(np.floor(xs))) == x0 and wrap(int(np.floor(np.float32(y)))) == y0
            checked += 1
    assert checked > 200


@pytest.mark.parametrize("beta", [0.05, 0.013])
def test_angular_fractions_follow_the_half_vector(orc, beta):
    """Flat normal (0, 0, 1): the shading frame is (x, y, z) itself, so the
    angular grid coordinate is h_x / beta - 1/2 with h = normalize(wi + wo)
    from the scene's directional view and light (fp64 here)."""
    gb = synth.random_gbuffer(6, 9, seed=32)
    nrm = gb.nrm.clone()
    nrm[..., 0] = 0.0
    nrm[..., 1] = 0.0
    nrm[..., 2] = 1.0
    gb = synth.GBuffer(gb.duv, gb.uvm, nrm, gb.pos, gb.mat)
    view, light = (0.3, -0.2, 0.9), (-0.45, 0.35, 0.8)
    sc = synth.SceneParams(seed=3, ndf="ggx", beta=beta, view_kind="directional", view=view,
                           lights=[synth.Light("directional", light, (1.0, 1.0, 1.0))])
    rec = _records(orc, gb, sc)
    wi = np.array(view) / np.linalg.norm(view)
    wo = np.array(light) / np.linalg.norm(light)
    h = (wi + wo) / np.linalg.norm(wi + wo)
    gx, gy = h[0] / beta - 0.5, h[1] / beta - 0.5
    act = rec["light_active"][:, 0] == 1
    assert act.sum() > 20
    r = rec[act, 0]
    assert np.all((r["afx"] >= 0) & (r["afx"] < 1) & (r["afy"] >= 0) & (r["afy"] < 1))
    np.testing.assert_allclose(r["cx0"] + r["afx"].astype(np.float64), gx, atol=2e-5 / beta * 0.05)
    np.testing.assert_allclose(r["cy0"] + r["afy"].astype(np.float64), gy, atol=2e-5 / beta * 0.05)
    assert np.all(r["cx0"] == math.floor(gx)) and np.all(r["cy0"] == math.floor(gy))


def test_pge1_is_the_closed_form_and_decides_T(orc):
    gb = synth.random_gbuffer(10, 13, seed=33)
    sc = synth.random_scene(33, n_lights=3)
    rec = _records(orc, gb, sc)
    r = rec[rec["light_active"] == 1]
    n, p, pge1, T = r["n"].astype(np.float64), r["p"].astype(np.float64)[:, None], r["pge1"].astype(np.float64), r["T"]
    live = (n > 0) & (p > 0)
    assert live.sum() > 200
    # closed form (Eq. 16) in fp64: 1 - (1 - p)^n = -expm1(n log1p(-p))
    with np.errstate(divide="ignore"):
        want = np.where(p >= 1, 1.0, -np.expm1(n * np.log1p(-np.minimum(p, 1 - 1e-16))))
    # the contract's fp32 log2 / exp2 polynomials: error relative to the
    # exponent (|n log2(1-p)|) plus fp32 rounding, and 1 - exp2(y) in fp32 is
    # absolute to an ulp of 1 (2^-23) when P>=1 is small
    err = np.abs(pge1 - want)
    tol = (4e-6 * np.maximum(want, 1e-30) + 2.0**-23
           + 1e-6 * np.abs(n * np.log2(np.maximum(1 - p, 1e-300))) * (1 - want))
    assert np.all(err[live] <= tol[live] + 1e-12), float(np.max((err - tol)[live]))
    # T = ceil(P>=1 2^23) exactly, and 0 with P>=1 = 0 where there are no trials
    assert np.array_equal(T[live], np.ceil(pge1[live] * 2.0**23).astype(np.uint32))
    assert np.all(pge1[~live] == 0) and np.all(T[~live] == 0)
