"""Quality battery for candidate per-draw hash designs (R-23, R-23b, §7
rejected variants, §12). CPU, numpy; no GPU needed.

A draw combines a texel seed hs (full lowbias32 of the texel's key) and an
angular-node seed ka (full lowbias32 of the node's key). The 4 angular nodes of
a texel must give nearly independent draws: for many random node cells,
measure between every pair of the 4 nodes (over 10^6 texel seeds)
  * the chi-square p-value of the 16 x 16 contingency of (gate bucket, gate
    bucket), (quantile bucket, quantile bucket), (gate, quantile) and of the
    quantile index's low bits,
  * the Pearson correlation of the gate indicators at P>=1 = 1/4 and of the
    quantiles (effect size; noise ~1e-3).
Candidates (ALU ops per draw in the kernel's draw loop, hash part only):
  current   draw_hash(hs + ka): t = x*C1; u = t ^ rotr(t, 15); y = u*C2;
            gate on y, index (y ^ y>>16)                          -- 5 ops
  shift15   the same with lowbias32's xor-shift u = t ^ t>>15
            (the round-1 design before R-23b)                    -- 5 ops
  xor_mul   (hs ^ ka) * C2                                        -- 2 ops
  premix    lowbias32-like: x = hs + ka; x ^= x>>16; then tail    -- 7 ops
  xor_tail  tail(hs ^ ka) (no pre-multiplication possible)        -- 6 ops
  u_index   current gate, index from u = t ^ (t>>15) bits 2..13   -- 4 ops

A second mode scans random node-seed offsets (`--node-pairs K`): for K random
pairs (ka0, ka1) of lowbias32 outputs, the worst chi-square p and Cramér's V
of the 4 contingencies between the two nodes' draws over 2^20 texel seeds,
for `current` and for the 7-op `premix` (a full lowbias32 of the sum).

usage: python tools/hash_quality.py [--n 1000000] [--cells 24] [--node-pairs 300]
"""
import argparse
import json

import numpy as np
from scipy import stats as st
from scipy.stats import norm

U = np.uint64
M = U(0xFFFFFFFF)
C1, C2 = U(0x7feb352d), U(0x846ca68b)


def lb(x):
    x = x & M
    x ^= x >> U(16); x = (x * C1) & M
    x ^= x >> U(15); x = (x * C2) & M
    return x ^ (x >> U(16))


def tail3(x, rotate=False):       # t = x*C1; u = t ^ t>>15 (or rotr 15); y = u*C2
    t = (x & M) * C1 & M
    u = t ^ ((((t >> U(15)) | (t << U(17))) & M) if rotate else (t >> U(15)))
    return (u * C2) & M, u


def rotr(t, k):
    return ((t >> U(k)) | (t << U(32 - k))) & M


def cand(name, hs, ka):
    """-> (y: gate word (bits 9..31), q: quantile index 0..4095)."""
    if name.startswith("rotm"):          # rotm:a:j -- u = t ^ (rotr(t,a) & ~(1 << j)): 2 ops, a bijection for odd a
        _, a, j = name.split(":")[:3]
        t = ((hs + ka) & M) * C1 & M
        u = t ^ (rotr(t, int(a)) & (M ^ U(1 << int(j))))
        y = (u * C2) & M
        return y, ((y ^ (y >> U(16))) >> U(2)) & U(4095)
    if name.startswith("rot3"):          # rot3:a:b -- t = x*C1; u = t ^ rotr(t,a) ^ rotr(t,b); y = u*C2 (bijective)
        _, a, b = name.split(":")[:3]
        t = ((hs + ka) & M) * C1 & M
        u = t ^ rotr(t, int(a)) ^ rotr(t, int(b))
        y = (u * C2) & M
        if name.endswith(":u"):          # quantile index from u (one op fewer)
            return y, (u >> U(2)) & U(4095)
        return y, ((y ^ (y >> U(16))) >> U(2)) & U(4095)
    if name == "current":
        y, _ = tail3(hs + ka, rotate=True)
        return y, ((y ^ (y >> U(16))) >> U(2)) & U(4095)
    if name == "shift15":
        y, _ = tail3(hs + ka)
        return y, ((y ^ (y >> U(16))) >> U(2)) & U(4095)
    if name == "xor_mul":
        y = ((hs ^ ka) * C2) & M
        return y, ((y ^ (y >> U(16))) >> U(2)) & U(4095)
    if name == "premix":
        x = (hs + ka) & M
        y, _ = tail3(x ^ (x >> U(16)))
        return y, ((y ^ (y >> U(16))) >> U(2)) & U(4095)
    if name == "xor_tail":
        y, _ = tail3(hs ^ ka)
        return y, ((y ^ (y >> U(16))) >> U(2)) & U(4095)
    if name == "u_index":
        y, u = tail3(hs + ka)
        return y, (u >> U(2)) & U(4095)
    raise ValueError(name)


OPS = {"rot3:15:7": 6, "current": 5, "shift15": 5, "xor_mul": 2, "premix": 7, "xor_tail": 6, "u_index": 4}


def battery(name, n, cells, seed=0):
    hs = lb(np.arange(n, dtype=U) * U(0x9e3779b1) + U(12345))
    z = norm.ppf((np.arange(4096) + 0.5) / 4096)
    rng = np.random.default_rng(seed)
    worst_p = {"gate-gate": 1.0, "quant-quant": 1.0, "gate-quant": 1.0, "quant-low-bits": 1.0}
    corr_g, corr_q = [], []
    for cx, cy in rng.integers(-500, 500, (cells, 2)):
        ka = [lb(U(((int(cx) + (j & 1)) * 0xcb1ab31f + (int(cy) + (j >> 1)) * 0x165667b1 + 0x27d4eb2f) & 0xFFFFFFFF))
              for j in range(4)]
        ys, qs = zip(*[cand(name, hs, k) for k in ka])
        for a in range(4):
            for b in range(a + 1, 4):
                for lab, (u, v) in (("gate-gate", (ys[a] >> U(28), ys[b] >> U(28))),
                                    ("quant-quant", (qs[a] >> U(8), qs[b] >> U(8))),
                                    ("gate-quant", (ys[a] >> U(28), qs[b] >> U(8))),
                                    ("quant-low-bits", (qs[a] & U(15), qs[b] & U(15)))):
                    tab = np.zeros((16, 16))
                    np.add.at(tab, (u.astype(np.int64), v.astype(np.int64)), 1)
                    worst_p[lab] = min(worst_p[lab], float(st.chi2_contingency(tab)[1]))
                ga = ((ys[a] >> U(9)) < U(1 << 21)).astype(float)
                gb = ((ys[b] >> U(9)) < U(1 << 21)).astype(float)
                corr_g.append(abs(np.corrcoef(ga, gb)[0, 1]))
                corr_q.append(abs(np.corrcoef(z[qs[a].astype(np.int64)], z[qs[b].astype(np.int64)])[0, 1]))
    return dict(ops=OPS.get(name, 5 if name.startswith('rotm') else (6 if not name.endswith(':u') else 5)), worst_chi2_p=worst_p, max_corr_gate=float(max(corr_g)),
                max_corr_quantile=float(max(corr_q)), pairs=len(corr_g))


def node_pair_scan(name, pairs, seed=3, n=1 << 20):
    """Random node-seed offsets: fraction of pairs whose draws are detectably
    dependent, and the largest effect size (Cramér's V; noise ~0.0013)."""
    hs = lb(np.arange(n, dtype=U) * U(0x9e3779b1) + U(99))
    rng = np.random.default_rng(seed)
    ps, vs, worst = [], [], []
    for _ in range(pairs):
        ka0, ka1 = [lb(U(int(v))) for v in rng.integers(0, 2 ** 32, 2)]
        y1, q1 = cand(name, hs, ka0)
        y2, q2 = cand(name, hs, ka1)
        best_p, best_v = 1.0, 0.0
        for u, v in ((y1 >> U(28), y2 >> U(28)), (q1 >> U(8), q2 >> U(8)), (y1 >> U(28), q2 >> U(8)),
                     (q1 & U(15), q2 & U(15))):
            tab = np.bincount((u * U(16) + v).astype(np.int64), minlength=256).reshape(16, 16)
            c, pv = st.chi2_contingency(tab)[:2]
            best_p = min(best_p, float(pv))
            best_v = max(best_v, float(np.sqrt(max(c - 225.0, 0.0) / n / 15)))
        ps.append(best_p)
        vs.append(best_v)
        worst.append((best_p, (int(ka1) - int(ka0)) * 0x7feb352d & 0xFFFFFFFF))
    ps, vs = np.array(ps), np.array(vs)
    return dict(pairs=pairs, frac_p_lt_1e3=float((ps < 1e-3).mean()), frac_expected=1 - (1 - 1e-3) ** 4,
                frac_p_lt_1e6=float((ps < 1e-6).mean()), max_cramers_v=float(vs.max()),
                median_cramers_v=float(np.median(vs)), worst_offsets_D=[f"{d:08x}" for _, d in sorted(worst)[:3]])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--cells", type=int, default=24)
    ap.add_argument("--node-pairs", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--names", default=None, help="comma-separated candidates (e.g. rot3:15:7,rot3:13:21:u)")
    a = ap.parse_args()
    if a.node_pairs:
        for name in (a.names.split(",") if a.names else ("current", "premix")):
            print(name, node_pair_scan(name, a.node_pairs), flush=True)
        return
    res = {}
    for name in (a.names.split(",") if a.names else OPS):
        res[name] = battery(name, a.n, a.cells)
        r = res[name]
        print(f"{name:9s} ops {r['ops']}  max|corr| gate {r['max_corr_gate']:.4f} quantile {r['max_corr_quantile']:.4f}  "
              "worst chi2 p " + " ".join(f"{k}={v:.1e}" for k, v in r["worst_chi2_p"].items()), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
