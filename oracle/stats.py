"""Statistical side of the oracle (fp64, numpy/scipy) -- TEST INFRASTRUCTURE ONLY.

These are the laws the paper states, written out plainly, used by the
``-m "not gpu"`` pin tests to check the C oracle against something other than
itself:

* the exact binomial law b(N, p) (its moments P:L162 footnote),
* the gated Gaussian law of Eq. 16-18 as a continuous-Phi pmf,
* the exact law of the gated draw under the fp32 contract, by enumerating all
  4096 quantile cells (reading R-2) through the C oracle's own count function,
* spatialised Bernoulli trials and stratified point sets (section 4.1,
  P:L449-460, Fig. 4),
* textbook smooth NDFs and their sampling routines for the brute-force facet
  check (BASELINE.json north-star check 1).
"""
from __future__ import annotations

import math

import numpy as np
from scipy import special, stats

from . import gate_params, gated_count, ZQ


# ---------------------------------------------------------------- binomial laws
def binom_pmf(n: int, p: float) -> np.ndarray:
    """Exact Binomial(n, p) pmf over k = 0..n (P:L154 b(N, p))."""
    k = np.arange(n + 1)
    return stats.binom.pmf(k, n, p)


def gated_pmf_analytic(n: float, p: float, kmax: int | None = None) -> np.ndarray:
    """Gated Gaussian approximation, continuous Phi (Eq. 16-18 + readings R-1..R-4):
    P(0) = 1 - P>=1 ; P(k) = P>=1 [Phi((k+1-m1)/s) - Phi((k-m1)/s)], k in [1, ceil n],
    the clamp folding the Gaussian tails into k = 1 and k = ceil(n)."""
    cap = int(math.ceil(n))
    kmax = cap if kmax is None else kmax
    pge1 = 1.0 - (1.0 - p) ** n
    mu = max(0.0, (n - 1.0) * p)
    s = math.sqrt(mu * (1.0 - p))
    m1 = 1.0 + mu
    out = np.zeros(kmax + 1)
    out[0] = 1.0 - pge1
    if s == 0.0:
        k = min(max(int(math.floor(m1)), 1), cap)
        out[k] += pge1
        return out
    cdf = lambda x: stats.norm.cdf((x - m1) / s)
    for k in range(1, cap + 1):
        lo = -np.inf if k == 1 else k
        hi = np.inf if k == cap else k + 1
        out[k] = pge1 * ((cdf(hi) if np.isfinite(hi) else 1.0) - (cdf(lo) if np.isfinite(lo) else 0.0))
    return out


def gated_pmf_enumerated(n: float, p: float):
    """Exact law of the contract's gated draw assuming an ideal hash: P(gate) =
    T / 2^23 and the count given the gate is a function of the quantile cell
    q = (h >> 2) & 4095 only (theta0 = (y >> 9) 2^-23 with y = h ^ (h >> 16), and
    z = Z[q]; the residual gate/quantile dependence is below 2^-18 and ignored
    here). Evaluated through
    the C oracle's own gate_params / gated_count for every q."""
    T, s, m1, cap = gate_params(n, p)
    # h = q << 2 has y = h (bits >= 16 are zero), y >> 9 < 2^7 <= T for T >= 128;
    # for tiny T pick the h with the same quantile cell and y >> 9 = 0
    counts = np.array([gated_count(q << 2, T, s, m1, cap) if T > 0 else 0 for q in range(ZQ)])
    kmax = int(max(cap, 1))
    pmf = np.zeros(kmax + 1)
    pg = T / float(1 << 23)
    pmf[0] = 1.0 - pg
    if T > 0:
        for k in range(1, kmax + 1):
            pmf[k] += pg * np.count_nonzero(counts == k) / ZQ
    return pmf, (T, s, m1, cap)


def pmf_mean(pmf: np.ndarray) -> float:
    return float(np.dot(np.arange(len(pmf)), pmf))


def total_variation(a: np.ndarray, b: np.ndarray) -> float:
    m = max(len(a), len(b))
    a = np.pad(a, (0, m - len(a)))
    b = np.pad(b, (0, m - len(b)))
    return 0.5 * float(np.abs(a - b).sum())


def chi2_gof(counts: np.ndarray, pmf: np.ndarray, min_expected: float = 5.0) -> float:
    """Chi-square goodness of fit p-value, pooling bins with small expectation."""
    counts = np.asarray(counts, float)
    m = max(len(counts), len(pmf))
    counts = np.pad(counts, (0, m - len(counts)))
    pmf = np.pad(np.asarray(pmf, float), (0, m - len(pmf)))
    M = counts.sum()
    exp = pmf * M
    obs_b, exp_b = [], []
    co = ce = 0.0
    for o, e in zip(counts, exp):
        co += o
        ce += e
        if ce >= min_expected:
            obs_b.append(co)
            exp_b.append(ce)
            co = ce = 0.0
    if ce > 0 or co > 0:
        if exp_b:
            obs_b[-1] += co
            exp_b[-1] += ce
        else:
            obs_b.append(co)
            exp_b.append(ce)
    obs_b, exp_b = np.array(obs_b), np.array(exp_b)
    if len(obs_b) < 2:
        return 1.0
    chi = float(((obs_b - exp_b) ** 2 / exp_b).sum())
    return float(stats.chi2.sf(chi, len(obs_b) - 1))


def chi2_two_sample(a: np.ndarray, b: np.ndarray) -> float:
    """Two-sample chi-square homogeneity p-value for integer samples."""
    lo = int(min(a.min(), b.min()))
    hi = int(max(a.max(), b.max()))
    ha = np.bincount(a - lo, minlength=hi - lo + 1).astype(float)
    hb = np.bincount(b - lo, minlength=hi - lo + 1).astype(float)
    keep = (ha + hb) >= 10
    rest = ~keep
    ha = np.append(ha[keep], ha[rest].sum())
    hb = np.append(hb[keep], hb[rest].sum())
    if ha[-1] + hb[-1] == 0:
        ha, hb = ha[:-1], hb[:-1]
    table = np.vstack([ha, hb])
    chi2, pval, _, _ = stats.chi2_contingency(table)
    return float(pval)


# ---------------------------------------------------------------- section 4.1
def stratified_points(m: int, rng: np.random.Generator) -> np.ndarray:
    """One uniformly jittered point per cell of an m x m grid on [0,1)^2 (P:L456
    'randomly jittered inside a regular grid')."""
    iy, ix = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    j = rng.random((m, m, 2))
    return np.stack([(ix + j[..., 0]) / m, (iy + j[..., 1]) / m], -1).reshape(-1, 2)


def spatialized_count(points: np.ndarray, success: np.ndarray, window) -> tuple[int, int]:
    """Spatialised Bernoulli trials: number of points x_i in the window
    A, and number of those whose mark succeeds (x_i in A and X_i < p)."""
    x0, y0, x1, y1 = window
    inside = (points[:, 0] >= x0) & (points[:, 0] < x1) & (points[:, 1] >= y0) & (points[:, 1] < y1)
    return int(inside.sum()), int((inside & success.astype(bool)).sum())


# ---------------------------------------------------------------- smooth NDFs (textbook)
def ndf_D(ndf: str, ax: float, ay: float, h: np.ndarray) -> np.ndarray:
    """Smooth anisotropic GGX / Beckmann D(h) for unit h in the local frame."""
    hx, hy, hz = h[..., 0], h[..., 1], h[..., 2]
    X = hx / ax
    Y = hy / ay
    if ndf == "ggx":
        q = X * X + Y * Y + hz * hz
        return 1.0 / (math.pi * ax * ay * q * q)
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(hz > 0, np.exp(-(X * X + Y * Y) / (hz * hz)) / (math.pi * ax * ay * hz ** 4), 0.0)


def sample_ndf_normals(ndf: str, alpha: float, n: int, rng: np.random.Generator) -> np.ndarray:
    """Isotropic normals with density D(m) (m.n) (inverse CDF of the slope law):
    GGX tan^2 = a^2 u/(1-u); Beckmann tan^2 = -a^2 ln(1-u)."""
    u1, u2 = rng.random(n), rng.random(n)
    if ndf == "ggx":
        t2 = alpha * alpha * u1 / (1.0 - u1)
    else:
        t2 = -alpha * alpha * np.log1p(-u1)
    ct = 1.0 / np.sqrt(1.0 + t2)
    st = np.sqrt(np.maximum(0.0, 1.0 - ct * ct))
    ph = 2 * math.pi * u2
    return np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1)


def smith_lambda_exact(ndf: str, alpha: float, cos_t: float) -> float:
    """Exact Smith Lambda: GGX (-1 + sqrt(1 + a^2 tan^2))/2; Beckmann
    (erf(a) - 1)/2 + exp(-a^2)/(2 a sqrt(pi)), a = 1/(alpha tan)."""
    tan2 = (1.0 - cos_t * cos_t) / (cos_t * cos_t)
    if ndf == "ggx":
        return 0.5 * (-1.0 + math.sqrt(1.0 + alpha * alpha * tan2))
    if tan2 == 0.0:
        return 0.0
    a = 1.0 / (alpha * math.sqrt(tan2))
    return 0.5 * (special.erf(a) - 1.0) + math.exp(-a * a) / (2.0 * a * math.sqrt(math.pi))
