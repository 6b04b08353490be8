"""Pins for S1 (footprint) and S2 (anisotropic lattice, Eq. 10/13,
P:L628-635, Fig. 6-7) against closed forms, SVD and the geometric
invariants the paper states (partition of unity, area conservation Eq. 10,
isotropy independence Fig. 6 caption, continuity, 9-tetrahedra tiling)."""
import math

import numpy as np
import pytest


def test_footprint_closed_forms(orc):
    P, r, psi, ok = orc.footprint([2.0, 0.0, 0.0, 1.0])     # J = diag(2, 1)
    assert ok and P == 2.0 and r == 2.0 and psi == 0.0
    P, r, psi, ok = orc.footprint([1.0, 0.0, 0.0, 1.0])     # J = I
    assert ok and P == 1.0 and r == 1.0
    P, r, psi, ok = orc.footprint([1.0 / 64, 0.0, 0.0, 1.0 / 64])   # C1
    assert ok and P == 2.0 ** -12 and r == 1.0 and psi == 0.0
    P, r, psi, ok = orc.footprint([0.0, 0.0, 0.0, 0.0])
    assert not ok
    P, r, psi, ok = orc.footprint([1.0, 0.0, 0.0, 3.0])     # major axis along v: phi = pi/2
    assert ok and r == 3.0 and abs(psi - 0.5) < 1e-7


def test_footprint_subnormal_anisotropy_is_isotropic(orc):
    """A near-isotropic footprint whose discriminant (a-c)^2/4 + b^2 is
    subnormal (C2 at 90 deg elevation, DESIGN R-30) reads as exactly isotropic,
    r = 1, with a finite orientation -- not the NaN the Newton steps of the
    contract rsqrt would give on a subnormal input."""
    s = np.float32(1.0691672e-02)
    P, r, psi, ok = orc.footprint([s, 0.0, 3.85e-21, -s])
    assert ok and r == 1.0 and 0.0 <= psi < 1.0
    assert abs(P - float(s) * float(s)) <= 1e-6 * P
    assert orc.atan2_turns(1e-45, 1e-45) == 0.0 and orc.atan2_turns(0.0, 0.0) == 0.0
    assert orc.atan2_turns(-2e-40, 3e-39) == 0.0


def test_footprint_vs_svd(orc):
    """P = s1 s2, r = s1/s2, psi = angle of the major singular vector / pi mod 1."""
    rng = np.random.default_rng(0)
    for _ in range(3000):
        J = rng.standard_normal((2, 2)) * 10.0 ** rng.uniform(-6, 1)
        J = J.astype(np.float32).astype(np.float64)
        U, S, Vt = np.linalg.svd(J)
        duv = [J[0, 0], J[1, 0], J[0, 1], J[1, 1]]
        P, r, psi, ok = orc.footprint(duv)
        assert ok
        assert abs(P - S[0] * S[1]) <= 1e-5 * S[0] * S[1] + 1e-6 * S[0] * S[0]
        rr = S[0] / S[1]
        if rr < 1e3:
            assert abs(r - rr) <= 1e-4 * rr
        if rr > 1.01:
            ang = math.atan2(U[1, 0], U[0, 0]) / math.pi % 1.0
            d = abs(psi - ang)
            assert min(d, 1 - d) < 1e-4 * max(1.0, 1.0 / (rr - 1.0))


def test_footprint_brute_force_ellipse(orc):
    """The ellipse {J (cos t, sin t)}: its farthest point lies along psi*pi and
    r = max radius / min radius (dense t sweep)."""
    rng = np.random.default_rng(1)
    t = np.linspace(0, 2 * np.pi, 200001)
    for _ in range(50):
        J = rng.standard_normal((2, 2)).astype(np.float32).astype(np.float64)
        pts = J @ np.stack([np.cos(t), np.sin(t)])
        rad = np.hypot(*pts)
        i = int(np.argmax(rad))
        P, r, psi, ok = orc.footprint([J[0, 0], J[1, 0], J[0, 1], J[1, 1]])
        assert abs(r - rad.max() / rad.min()) < 1e-4 * r
        if r > 1.05:
            ang = math.atan2(pts[1, i], pts[0, i]) / math.pi % 1.0
            d = abs(psi - ang)
            assert min(d, 1 - d) < 1e-3


# ------------------------------------------------------------------ lattice
def _vertex_field(ls, lr, jo):
    """A random-but-fixed scalar per lattice vertex (to probe continuity)."""
    h = (ls * 73856093) ^ (lr * 19349663) ^ (jo * 83492791)
    return ((h * 2654435761) % 2 ** 32) / 2 ** 32


def _interp(orc, P, r, psi, K=8):
    ls, lr, jo, w, _ = orc.lattice(P, r, psi, K)
    return sum(wi * _vertex_field(a, b, c) for a, b, c, wi in zip(ls, lr, jo, w)), (ls, lr, jo, w)


def test_partition_area_and_sign(orc):
    rng = np.random.default_rng(2)
    for _ in range(20000):
        P = float(np.float32(2.0 ** rng.uniform(-40, 30)))
        r = float(np.float32(2.0 ** rng.uniform(0, 9)))
        psi = float(np.float32(rng.random()))
        ls, lr, jo, w, fl = orc.lattice(P, r, psi)
        w = np.array(w, np.float64)
        assert w.min() >= -1e-7
        assert abs(w.sum() - 1.0) < 2e-6
        # Eq. 10 / reading R-14: sum_i w_i * area_i == P (area conservation)
        area = sum(wi * 2.0 ** a for wi, a in zip(w, ls))
        assert abs(area - P) <= 4e-6 * P
        # Eq. 13: top-level share is (P - Plow)/(Phigh - Plow)
        e = math.floor(math.log2(P))
        assert set(ls) <= {e, e + 1}
        top = sum(wi for wi, a in zip(w, ls) if a == e + 1)
        assert abs(top - (P / 2.0 ** e - 1.0)) < 2e-6
        # at most 4 distinct grids, nonzero weights on distinct keys
        keys = [(a, b, c) for a, b, c, wi in zip(ls, lr, jo, w) if wi > 0]
        assert len(keys) == len(set(keys))
        if r <= 256:
            assert fl == 0


def test_linear_precision_ratio_and_orientation(orc):
    """Barycentric interpolation reproduces the lattice coordinates: sum w_i t_r,i
    = t_r and (ring >= 1) sum w_i a_i = a, with the pentagon's vertex positions
    A00=(0,0) A01=(0,1) A10=(1,0) A11=(1,1/2) A12=(1,1) (reading R-11)."""
    rng = np.random.default_rng(3)
    for _ in range(20000):
        er = int(rng.integers(0, 8))
        tr = float(np.float32(rng.random()))
        r = float(np.float32(2.0 ** er * (1 + tr)))
        tr = r / 2.0 ** er - 1.0
        if not (r < 256):
            continue
        psi = float(np.float32(rng.random()))
        P = float(np.float32(2.0 ** rng.uniform(-20, 5)))
        ls, lr, jo, w, _ = orc.lattice(P, r, psi)
        got_tr = sum(wi for wi, b in zip(w, lr) if b == er + 1)
        assert abs(got_tr - tr) < 3e-6
        if er >= 1:
            A = psi * 2 ** er
            j = math.floor(A)
            a = A - j
            acc = 0.0
            for wi, b, c in zip(w, lr, jo):
                if b == er:
                    av = (c - j) % (2 ** er)
                else:
                    av = ((c - 2 * j) % (2 ** (er + 1))) / 2.0
                acc += wi * av
            assert abs(acc - a) < 4e-6


def test_vertex_reproduction(orc):
    """At a lattice vertex (P = 2^e, r = 2^k, psi = j/2^k) the weight is one-hot."""
    for e in (-20, -3, 0, 7):
        for k in range(0, 8):
            for j in range(0, 2 ** k, max(1, 2 ** k // 4)):
                ls, lr, jo, w, _ = orc.lattice(2.0 ** e, 2.0 ** k, j / 2 ** k)
                nz = [(a, b, c) for a, b, c, wi in zip(ls, lr, jo, w) if wi != 0]
                assert nz == [(e, k, j)], (e, k, j, ls, lr, jo, w)
                assert max(w) == 1.0


def test_isotropic_footprint_ignores_orientation(orc):
    """r = 1: 'a single isotropic grid accounts for orientation'."""
    rng = np.random.default_rng(4)
    nz = lambda L: sorted((a, b, c, wi) for a, b, c, wi in zip(*L[:4]) if wi != 0)
    for _ in range(2000):
        P = float(np.float32(2.0 ** rng.uniform(-30, 10)))
        ref = nz(orc.lattice(P, 1.0, 0.0))
        assert all(b == 0 and c == 0 for _, b, c, _ in ref)
        for psi in rng.random(3):
            assert nz(orc.lattice(P, 1.0, float(np.float32(psi)))) == ref


@pytest.mark.parametrize("axis", ["scale", "ratio", "orient", "wrap"])
def test_continuity_across_cell_faces(orc, axis):
    """Interpolated vertex fields are continuous across LOD, ratio-ring, sector,
    pentagon-triangle and wrap boundaries (artifact-free blending)."""
    rng = np.random.default_rng({"scale": 5, "ratio": 6, "orient": 7, "wrap": 8}[axis])
    for _ in range(400):
        P = float(np.float32(2.0 ** rng.uniform(-20, 5)))
        r = float(np.float32(2.0 ** rng.uniform(0.01, 7.9)))
        psi = float(np.float32(rng.uniform(0.001, 0.999)))
        if axis == "scale":
            e = math.floor(math.log2(P))
            pts = [(float(np.float32(2.0 ** e * (1 + d))), r, psi) for d in (-3e-6, 0.0, 3e-6)]
            pts[0] = (float(np.nextafter(np.float32(2.0 ** e), np.float32(0))), r, psi)
        elif axis == "ratio":
            k = int(rng.integers(1, 8))
            pts = [(P, float(np.nextafter(np.float32(2.0 ** k), np.float32(0))), psi), (P, 2.0 ** k, psi)]
        elif axis == "orient":
            k = math.floor(math.log2(r)) + 1
            j = int(rng.integers(0, 2 ** k))
            b = np.float32(j / 2 ** k + 1e-9)
            pts = [(P, r, float(np.nextafter(np.float32(j / 2 ** k), np.float32(0)))), (P, r, float(np.float32(j / 2 ** k)))]
            if j == 0:
                pts[0] = (P, r, float(np.nextafter(np.float32(1.0), np.float32(0))))
        else:
            pts = [(P, r, float(np.nextafter(np.float32(1.0), np.float32(0)))), (P, r, 0.0)]
        vals = [_interp(orc, *pt)[0] for pt in pts]
        assert max(vals) - min(vals) < 1e-4, (axis, pts, vals)
    # interior faces: random points and tiny perturbations in all coordinates
    for _ in range(3000):
        P = float(np.float32(2.0 ** rng.uniform(-20, 5)))
        r = float(np.float32(2.0 ** rng.uniform(0.0, 7.99)))
        psi = float(np.float32(rng.random()))
        f0, _ = _interp(orc, P, r, psi)
        f1, _ = _interp(orc, float(np.float32(P * (1 + 1e-6))), float(np.float32(r * (1 + 1e-6))),
                        float(np.float32(psi + 1e-6)) % 1.0)
        assert abs(f1 - f0) < 1e-3


def test_nine_tetrahedra_tile_the_prism(orc):
    """Each triangular prism splits into 3 tetrahedra of equal volume; triangles
    T0, T2 have area 1/4 and T1 area 1/2, so the 9 tetrahedra occupy 1/12,1/12,
    1/12, 1/6,1/6,1/6, 1/12,1/12,1/12 of the cell (Fig. 7). Identify the
    tetrahedron by which pentagon vertices carry weight and which staircase
    step is active; count uniform samples."""
    rng = np.random.default_rng(9)
    er = 3
    counts = {}
    M = 60000
    for _ in range(M):
        ts, tr, a = rng.random(3)
        P = float(np.float32(2.0 ** -5 * (1 + ts)))
        r = float(np.float32(2.0 ** er * (1 + tr)))
        psi = float(np.float32((5 + a) / 2 ** er))
        ls, lr, jo, w, _ = orc.lattice(P, r, psi)
        tr32 = r / 2.0 ** er - 1
        a32 = psi * 2 ** er - 5
        tri = 0 if a32 <= tr32 / 2 else (2 if a32 >= 1 - tr32 / 2 else 1)
        n_top = sum(1 for l in ls if l == -4)
        counts[(tri, n_top)] = counts.get((tri, n_top), 0) + 1
    expect = {(0, 1): 1 / 12, (0, 2): 1 / 12, (0, 3): 1 / 12, (1, 1): 1 / 6, (1, 2): 1 / 6, (1, 3): 1 / 6,
              (2, 1): 1 / 12, (2, 2): 1 / 12, (2, 3): 1 / 12}
    assert set(counts) == set(expect)
    for key, frac in expect.items():
        sd = math.sqrt(frac * (1 - frac) / M)
        assert abs(counts[key] / M - frac) < 5 * sd, (key, counts[key] / M, frac)


def test_c1_reduces_to_a_single_grid(orc):
    """C1: P = 2^-12, r = 1 -> grid (ls, lr, jo) = (-12, 0, 0) with weight 1."""
    ls, lr, jo, w, _ = orc.lattice(2.0 ** -12, 1.0, 0.0)
    nz = [(a, b, c, wi) for a, b, c, wi in zip(ls, lr, jo, w) if wi != 0]
    assert nz == [(-12, 0, 0, 1.0)]


def test_ratio_clamp(orc):
    ls, lr, jo, w, fl = orc.lattice(1.0, 1e6, 0.3)
    assert fl == 4 and max(lr) == 8 and abs(sum(w) - 1) < 1e-6
    assert all(b == 8 for b, wi in zip(lr, w) if wi > 0)


@pytest.mark.parametrize("K", [1, 2, 3, 5, 7])
def test_lattice_smaller_max_ratio_level(orc, K):
    """K < 8 (the ABI's max_ratio_level): ratio levels 0..K, orientation
    indices below 2^lr, partition of unity and area conservation everywhere,
    the clamp flag exactly when r > 2^K, and any r >= 2^K lattices like r = 2^K
    (reading R-9; clamp C-25)."""
    rng = np.random.default_rng(40 + K)
    for _ in range(4000):
        P = float(np.float32(2.0 ** rng.uniform(-30, 10)))
        r = float(np.float32(2.0 ** rng.uniform(0, K + 2)))
        psi = float(np.float32(rng.random()))
        ls, lr, jo, w, fl = orc.lattice(P, r, psi, K)
        w = np.array(w, np.float64)
        assert w.min() >= -1e-7 and abs(w.sum() - 1) < 2e-6
        assert abs(sum(wi * 2.0 ** a for wi, a in zip(w, ls)) - P) <= 4e-6 * P
        for b, c, wi in zip(lr, jo, w):
            if wi > 0:
                assert 0 <= b <= K and 0 <= c < 2 ** b
        assert (fl == 4) == (r > 2.0 ** K)
        if r >= 2.0 ** K:
            assert orc.lattice(P, r, psi, K)[:4] == orc.lattice(P, 2.0 ** K, psi, K)[:4]


def test_call_budget_is_48_draws_whatever_the_footprint(orc):
    """SURVEY 8c-2 "call budget": every active (pixel, light) evaluates
    exactly 4 grids x 3 texels x 4 nodes = 48 draws, whatever the footprint's
    size or anisotropy: the 48 draw words of a record are all computed (no
    zero left from the zero-filled record beyond chance); the 12 draws of each
    weighted slot are distinct (slots merged at ring 0 keep zero weight and
    repeat the key of the slot they merged into)."""
    from paper_2306_05051_b200 import synth
    gb = synth.random_gbuffer(40, 50, seed=48)
    sc = synth.random_scene(48, n_lights=2)
    _, fl, rec = orc.eval(gb, sc, debug=True)
    active = rec["light_active"] == 1
    assert active.sum() > 500
    h = rec["hash"][active]
    assert h.shape[1] == 48
    nonzero = (h != 0).sum(1)
    assert nonzero.min() >= 47
    w = rec["w"][active]
    for row, ww in zip(h, w):
        words = [x for s in range(4) if ww[s] > 0 for x in row[s * 12:(s + 1) * 12].tolist()]
        assert len(set(words)) >= len(words) - 1
