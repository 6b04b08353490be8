"""Pins for S6/S7: the gated Gaussian binomial approximation (Eq. 16-18,
P:L986-1000) under the contract's quantised uniforms (readings R-1..R-4, R-23)."""
import math

import numpy as np
import pytest

from oracle import stats


def test_special_cases(orc):
    assert orc.gate_params(10.0, 0.0)[0] == 0            # p = 0 -> never
    assert orc.gate_params(0.0, 0.5)[0] == 0             # n = 0 -> never
    T, s, m1, cap = orc.gate_params(5.0, 1.0)            # p = 1 -> always, count = n
    assert T == 2 ** 23 and s == 0.0 and m1 == 5.0 and cap == 5.0
    for h in (0, 123456789, 2 ** 32 - 1):
        assert orc.gated_count(h, T, s, m1, cap) == 5
    T, s, m1, cap = orc.gate_params(64.0, 0.5)
    assert m1 == 32.5 and abs(s - math.sqrt(15.75)) < 1e-6


@pytest.mark.parametrize("p", [1e-6, 0.01, 0.034, 0.3, 0.5, 0.9, 0.999])
def test_single_trial_gate_probability_is_p(orc, p):
    """n = 1: P>=1 = 1 - (1-p)^1 = p (Eq. 16); the count is 0 or 1."""
    T, s, m1, cap = orc.gate_params(1.0, p)
    assert abs(T / 2 ** 23 - p) <= 2 ** -23 + 2e-7 * p
    assert s == 0.0 and cap == 1.0
    pmf, _ = stats.gated_pmf_enumerated(1.0, p)
    assert len(pmf) == 2


@pytest.mark.parametrize("n", [0.3, 1.0, 4.0, 16.0, 24.4140625, 64.0, 1000.0, 1e5])
@pytest.mark.parametrize("p", [0.001, 0.05, 0.5, 0.95])
def test_zero_class_is_one_minus_p_to_the_n(orc, n, p):
    """P(count = 0) = (1 - p)^n by construction of the gate (Eq. 16)."""
    pmf, (T, s, m1, cap) = stats.gated_pmf_enumerated(n, p)
    assert abs(pmf[0] - (1 - p) ** n) <= 2 ** -23 + 1e-6 * max(1e-30, (1 - p) ** n) + 3e-7


@pytest.mark.parametrize("n,p", [(4, 0.3), (16, 0.3), (24.4140625, 0.034), (64, 0.05), (64, 0.5),
                                 (200.5, 0.2), (1e4, 0.034)])
def test_enumerated_law_matches_gated_gaussian(orc, n, p):
    """The contract's exact law (4096 quantile cells) equals Eq. 18's gated
    Gaussian with a continuous Phi up to the 1/4096 quantisation per bin edge."""
    pmf_e, _ = stats.gated_pmf_enumerated(n, p)
    pmf_a = stats.gated_pmf_analytic(n, p)
    nbins = int(np.count_nonzero(pmf_a > 1e-9))
    assert stats.total_variation(pmf_e, pmf_a) <= 1e-6 + nbins / 4096.0


def test_tv_to_exact_binomial_is_reported_not_asserted(orc):
    """the paper's sampler is not the exact binomial; the TV
    distances it quotes (continuous Phi) are reproduced here to 1e-3."""
    for (n, p), tv in {(2, 0.5): 0.131, (4, 0.95): 0.471, (16, 0.3): 0.062, (64, 0.5): 0.004}.items():
        assert abs(stats.total_variation(stats.gated_pmf_analytic(n, p), stats.binom_pmf(n, p)) - tv) < 1.5e-3


def test_large_n_mean_has_the_floor_bias(orc):
    """For large n the gated mean tends to n p + 1/2 - p (floor of 1 + N(mu, s)):
    +0.14 % at n = 1e4, p = 0.034."""
    pmf, _ = stats.gated_pmf_enumerated(1e4, 0.034)
    m = stats.pmf_mean(pmf)
    assert abs(m - (1e4 * 0.034 + 0.5 - 0.034)) < 0.05
    assert abs(m / (1e4 * 0.034) - 1.0014) < 2e-4


def test_hashed_draws_follow_the_enumerated_law(orc):
    """Draws made through the oracle's hash (C1 mirror: slot n = 24.414, p =
    0.034) follow the enumerated law (chi-square), i.e. the hash's gate bits
    and quantile bits behave as independent uniforms (reading R-23)."""
    from paper_2306_05051_b200 import synth
    fr = synth.c1("ggx", "mirror")
    _, _, rec = orc.eval(fr.gbuf, fr.scene, debug=True)
    r = rec[:, 0]
    h = r["hash"][:, :12].ravel()
    c = r["count"][:, :12].ravel()
    _, first = np.unique(h, return_index=True)          # each (texel, node) once
    c = c[first].astype(np.int64)
    assert len(c) > 10000
    pmf, (T, *_rest) = stats.gated_pmf_enumerated(float(r["n"][0, 0]), float(r["p"][0]))
    assert T == r["T"][0, 0]
    pv = stats.chi2_gof(np.bincount(c, minlength=len(pmf)), pmf)
    assert pv > 1e-3, pv
