"""Pins for S3: the anisotropic grid transform (Eq. 12, reading
R-14) and the simplex surface grid (Fig. 8 shear P:L882)."""
import math

import numpy as np


def _inverse_map(x, y, ls, lr, jo):
    """fp64 inverse of reading R-14: uv = R(-phi) diag(sqrt(A R), sqrt(A/R)) (x, y)."""
    A, Rr = 2.0 ** ls, 2.0 ** lr
    phi = jo * 2 ** (8 - lr) * math.pi / 256
    xs, ys = x * math.sqrt(A * Rr), y * math.sqrt(A / Rr)
    return (math.cos(phi) * xs - math.sin(phi) * ys, math.sin(phi) * xs + math.cos(phi) * ys)


def test_texel_is_footprint_shaped_rectangle(orc):
    """A unit texel of grid (ls, lr, jo) is a sqrt(AR) x sqrt(A/R) rectangle of
    area A = 2^ls whose long side points along phi_j (one texel per footprint,
    P:L618 'align the texels with the projected pixel footprint')."""
    rng = np.random.default_rng(0)
    for _ in range(500):
        ls, lr = int(rng.integers(-24, 4)), int(rng.integers(0, 9))
        jo = int(rng.integers(0, 2 ** lr))
        corners = [np.array(_inverse_map(x, y, ls, lr, jo)) for x, y in ((0, 0), (1, 0), (0, 1))]
        e1, e2 = corners[1] - corners[0], corners[2] - corners[0]
        assert abs(abs(e1[0] * e2[1] - e1[1] * e2[0]) - 2.0 ** ls) < 1e-9 * 2.0 ** ls
        assert abs(np.linalg.norm(e1) / np.linalg.norm(e2) - 2.0 ** lr) < 1e-9 * 2.0 ** lr
        # forward map (oracle, fp32) of a uv point and of the point moved by e1
        u, v = rng.random(2) * 0.5
        x0, y0 = orc.grid_uv(float(u), float(v), ls, lr, jo)
        x1, y1 = orc.grid_uv(float(u + e1[0]), float(v + e1[1]), ls, lr, jo)
        tol = 4e-6 * max(1.0, abs(x0), abs(y0))
        assert abs((x1 - x0) - 1.0) < tol and abs(y1 - y0) < tol * 2.0 ** lr


def test_c1_grid_is_pixel_lattice(orc):
    """C1: grid (-12, 0, 0) scales uv = pixel/64 by 2^6 -> uv' = pixel index exactly."""
    for px in range(64):
        for py in (0, 1, 17, 63):
            x, y = orc.grid_uv(px / 64.0, py / 64.0, -12, 0, 0)
            assert x == px and y == py


def test_simplex_partition_one_hot_and_linear_precision(orc):
    rng = np.random.default_rng(1)
    for _ in range(20000):
        x, y = (rng.random(2) - 0.5) * 2000
        x, y = float(np.float32(x)), float(np.float32(y))
        lx, ly, b = orc.simplex(x, y)
        b = np.array(b, np.float64)
        assert b.min() >= 0.0 and abs(b.sum() - 1.0) < 1e-6
        # sum b_k * vertex = point in sheared lattice coords (x + y/2, y)
        xs = np.float32(x) + np.float32(0.5) * np.float32(y)
        assert abs(float(np.dot(b, lx)) - float(xs)) < 1e-4
        assert abs(float(np.dot(b, ly)) - y) < 1e-4
    for ix in range(-3, 4):
        for iy in range(-3, 4):
            # lattice point (ix, iy) in sheared coords is (ix - iy/2, iy) in grid space
            lx, ly, b = orc.simplex(ix - iy / 2.0, float(iy))
            assert b[0] == 1.0 and (lx[0], ly[0]) == (ix, iy)


def test_simplex_continuity(orc):
    """Interpolated lattice fields are continuous across triangle edges."""
    rng = np.random.default_rng(2)
    val = lambda i, j: ((i * 73856093 ^ j * 19349663) * 2654435761 % 2 ** 32) / 2 ** 32
    f = lambda x, y: sum(bk * val(i, j) for i, j, bk in zip(*orc.simplex(x, y)))
    for _ in range(5000):
        x, y = (rng.random(2) - 0.5) * 100
        d = 1e-4
        assert abs(f(float(x), float(y)) - f(float(x + d), float(y + d * 0.7))) < 5e-3


def test_c1_simplex_pattern(orc):
    """C1 pixel lattice: even rows sit on lattice points (beta = (1,0,0)); odd
    rows sit at the midpoint of a lattice edge (beta = (1/2, 1/2, 0))."""
    for px in range(0, 64, 7):
        for py in range(0, 8):
            lx, ly, b = orc.simplex(float(px), float(py))
            if py % 2 == 0:
                assert b == [1.0, 0.0, 0.0] and (lx[0], ly[0]) == (px + py // 2, py)
            else:
                assert sorted(b) == [0.0, 0.5, 0.5]
