"""Spatial draw-hash battery (R-23b, profiles/r1_hash_quality.md):
candidate TEXEL seeds hs = f(lattice key) for the draw hash
draw_hash(hs + ka_j). Over 2000^2 texels of one grid, compares each texel's
draw with its lattice neighbours (x+1, y+1, diagonal), with another angular
node, and with grids whose key differs by 1 / 512 / 8192; 16x16 chi-square
contingencies of gate / quantile buckets (5 per pair) and |correlation|.
Candidates: current (hs = lowbias32(key), 9 ops with the pre-multiplication),
mix1 (x ^= x >> 16; x *= C: 3 ops), none (hs = key: 1 op).

usage: python tools/hash_quality_spatial.py <current|mix1|none> <seed> <trials>
"""
import sys

import numpy as np
from scipy import stats as st

U = np.uint64
M = U(0xFFFFFFFF)
C1, C2 = U(0x7feb352d), U(0x846ca68b)
A, B, Cc = U(0x9e3779b1), U(0x8da6b343), U(0xd8163841)     # key, lx, ly multipliers (DESIGN §4.3 S4)


def lb(x):
    x = x & M
    x ^= x >> U(16); x = (x * C1) & M
    x ^= x >> U(15); x = (x * C2) & M
    return x ^ (x >> U(16))


def mix1(x):
    x = x & M
    x ^= x >> U(16)
    return (x * U(0x2c1b3c6d)) & M


def draw(x):
    """the product's draw hash: gate word y and quantile index"""
    t = (x & M) * C1 & M
    u = t ^ (((t >> U(15)) | (t << U(17))) & M)
    y = (u * C2) & M
    return y, ((y ^ (y >> U(16))) >> U(2)) & U(4095)


SEED = {"current": lb, "none": lambda v: v & M, "mix1": mix1}


def chi2p(u, v):
    tab = np.bincount((u * U(16) + v).astype(np.int64), minlength=256).reshape(16, 16)
    return st.chi2_contingency(tab)[1]


def main():
    cand, seed, trials = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    rng = np.random.default_rng(seed)
    n = 2000
    iy, ix = np.meshgrid(np.arange(n, dtype=U), np.arange(n, dtype=U), indexing="ij")
    ix, iy = ix.ravel(), iy.ravel()
    allp, corr = {}, {}
    for _ in range(trials):
        so = U(int(rng.integers(0, 2 ** 32)))
        key = U(int(rng.integers(0, 2 ** 20)))
        ka = [lb(U(int(v))) for v in rng.integers(0, 2 ** 32, 4)]
        ox, oy = U(int(rng.integers(0, 2 ** 31))), U(int(rng.integers(0, 2 ** 31)))

        def d(dx, dy, dk, j):
            lin = (so + (key + U(dk)) * A + (ix + ox + U(dx)) * B + (iy + oy + U(dy)) * Cc) & M
            return draw((SEED[cand](lin) + ka[j]) & M)
        y1, q1 = d(0, 0, 0, 0)
        for nm, (y2, q2) in {"tx": d(1, 0, 0, 0), "ty": d(0, 1, 0, 0), "td": d(1, 1, 0, 0), "node": d(0, 0, 0, 1),
                             "key1": d(0, 0, 1, 0), "key512": d(0, 0, 512, 0), "key8192": d(0, 0, 8192, 0)}.items():
            for a, b in ((y1 >> U(28), y2 >> U(28)), (q1 >> U(8), q2 >> U(8)), (y1 >> U(28), q2 >> U(8)),
                         (q1 & U(15), q2 & U(15)), ((q1 >> U(4)) & U(15), (q2 >> U(4)) & U(15))):
                allp.setdefault(nm, []).append(chi2p(a, b))
            g1 = (y1 >> U(9) < U(2 ** 21)).astype(float)
            g2 = (y2 >> U(9) < U(2 ** 21)).astype(float)
            corr[nm] = max(corr.get(nm, 0.0), abs(np.corrcoef(g1, g2)[0, 1]),
                           abs(np.corrcoef(q1.astype(float), q2.astype(float))[0, 1]))
    ps = np.concatenate([np.array(v) for v in allp.values()])
    print(cand, "tests", len(ps), "min p %.1e" % ps.min(), "frac<0.01 %.3f" % (ps < 0.01).mean(),
          "KS %.3f" % st.kstest(ps, "uniform").pvalue,
          " ".join(f"{k}:{min(v):.0e}/{corr[k]:.4f}" for k, v in allp.items()))


if __name__ == "__main__":
    main()
