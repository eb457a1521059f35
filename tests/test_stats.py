"""stats.hpp diagnostics (paper_1912_12607_b200/stats.py): MLE fits, CDFs and the
KS statistic against scipy.stats (the checker), histogram rule, snapshot
summary; the device histogram (i8t_histogram) against the host rule on a GPU."""
import math

import numpy as np
import pytest
import torch
from scipy import stats as sps

from paper_1912_12607_b200 import stats as S


def _heavy(n=4000, seed=0):
    rng = np.random.default_rng(seed)
    return (rng.standard_t(3.0, n) * 2e-4 + 1e-5).astype(np.float32)


def test_cdfs_match_scipy():
    for x in (-3.0, -0.7, 0.0, 0.2, 1.5, 4.0):
        assert S.gaussian_cdf(x, 0.3, 1.7) == pytest.approx(sps.norm.cdf(x, 0.3, 1.7), rel=1e-13, abs=1e-15)
        assert S.laplace_cdf(x, 0.3, 1.7) == pytest.approx(sps.laplace.cdf(x, 0.3, 1.7), rel=1e-13, abs=1e-15)
        for nu in (1.0, 2.5, 7.0, 60.0):
            assert S.student_t_cdf(x, 0.3, 1.7, nu) == pytest.approx(sps.t.cdf(x, nu, 0.3, 1.7), rel=1e-10, abs=1e-13)


def test_gaussian_and_laplace_mle_are_the_closed_forms():
    x = _heavy().astype(np.float64)
    g = S.fit_mle(S.DistFamily.GAUSSIAN, x)
    mu, sd = sps.norm.fit(x)
    assert g.location == pytest.approx(mu, rel=1e-12) and g.scale == pytest.approx(sd, rel=1e-12)
    lap = S.fit_mle(S.DistFamily.LAPLACE, x)
    assert lap.location == pytest.approx(np.median(x), rel=1e-12)
    assert lap.scale == pytest.approx(np.mean(np.abs(x - np.median(x))), rel=1e-12)


def test_student_t_fit_recovers_heavy_tail_and_maximises_likelihood():
    x = _heavy(6000, 1).astype(np.float64)
    t = S.fit_mle(S.DistFamily.STUDENT_T, x)
    assert 2.0 <= t.nu <= 5.0
    ll = np.sum(sps.t.logpdf(x, t.nu, t.location, t.scale))
    for dnu in (-1.0, 1.0):  # the chosen nu beats its grid neighbours at their own EM optimum
        nu = t.nu + dnu
        mu, sig, _ = S._student_t_em(x, nu)
        assert ll >= np.sum(sps.t.logpdf(x, nu, mu, sig)) - 1e-6


def test_ks_statistic_matches_scipy_and_rejects_gaussian_on_heavy_tails():
    x = _heavy(3000, 2)
    for fam in S.DistFamily:
        f = S.fit_and_test(fam, x)
        ref = sps.kstest(x.astype(np.float64), lambda v: np.array([S.dist_cdf(f, float(u)) for u in np.atleast_1d(v)]))
        assert f.ks == pytest.approx(ref.statistic, rel=1e-12)
        assert f.critical == pytest.approx(1.358 / math.sqrt(x.size))
    assert S.fit_and_test(S.DistFamily.GAUSSIAN, x).rejected()
    assert not S.fit_and_test(S.DistFamily.STUDENT_T, x).rejected()


def test_ks_requires_100_samples_and_variance():
    with pytest.raises(ValueError):
        S.ks_statistic(np.ones(50, np.float32), S.DistFit(S.DistFamily.GAUSSIAN, 0.0, 1.0))
    with pytest.raises(ValueError):
        S.ks_statistic(np.ones(200, np.float32), S.DistFit(S.DistFamily.GAUSSIAN, 1.0, 1.0))


def test_host_histogram_rule_and_summary():
    x = np.array([-2.0, -1.0, 0.0, 0.5, 2.0, np.nan, np.inf], np.float32)
    h = S.make_histogram(x, bins=4, iter=7, layer="l")
    assert (h.lo, h.hi, h.iter, h.layer) == (-2.0, 2.0, 7, "l")
    assert h.counts == [1, 1, 2, 1] and h.total() == 5  # v == hi lands in the last bin; non-finite skipped
    z = S.make_histogram(np.zeros(10, np.float32), bins=2)
    assert (z.lo, z.hi, z.counts) == (-1.0, 1.0, [0, 10])
    s = S.summarize_samples("l", 3, np.array([-1.0, 2.0, 0.0], np.float32))
    assert (s.min, s.max, s.range, s.max_abs) == (-1.0, 2.0, 3.0, 2.0)
    assert s.kurtosis_proxy == pytest.approx((1 + 16) / 3 / ((1 + 4) / 3) ** 2)


@pytest.mark.gpu
@pytest.mark.parametrize("n,bins", [(1, 8), (1000, 64), (3_000_001, 257), (2_000_000, 4096)])
def test_device_histogram_equals_host_rule(n, bins):
    rng = np.random.default_rng(n)
    x = (rng.laplace(0, 1e-3, n)).astype(np.float32)
    if n > 10:
        x[rng.integers(0, n, 5)] = np.nan
        x[rng.integers(0, n, 3)] = -np.inf
    h = S.make_histogram(torch.from_numpy(x).cuda(), bins=bins)
    lo, hi, counts = S._host_histogram(x, bins)
    assert (h.lo, h.hi) == (lo, hi)
    assert h.counts == counts.tolist()
    zh = S.make_histogram(torch.zeros(100, device="cuda"), bins=4)
    assert (zh.lo, zh.hi, zh.counts) == (-1.0, 1.0, [0, 0, 100, 0])
