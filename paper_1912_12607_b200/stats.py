"""Distribution diagnostics of gradients / activations: the API the reference
declares in `proj/core/include/i8t/stats.hpp` (no implementation ships with
it).  Histogram (`make_histogram`, :11-23) runs on the device for CUDA tensors
(`i8t_histogram`, csrc/dsgc.cu); the maximum-likelihood fits, the CDFs, the
Kolmogorov-Smirnov statistic and the snapshot summary (:25-64) are host-side
float64 arithmetic on the sample array -- diagnostics for the trace, off the
training hot path.

Definitions where the header leaves them open (documented, tested in
tests/test_stats.py):
* histogram bin of v: floor((v - lo) / (hi - lo) * bins) in double, clamped to
  [0, bins - 1], over [-m, m], m = max|x| of the finite samples ([-1, 1] when m = 0);
  non-finite samples are not counted;
* Gaussian MLE: mean and population standard deviation; Laplace MLE: median
  and mean absolute deviation from it; Student-t: nu on the grid 1..100, for
  each nu the location/scale by EM (iteratively reweighted), the nu of
  largest log-likelihood kept;
* KS: sup over the sorted samples of max(i/N - F(x_i), F(x_i) - (i-1)/N);
  critical value 1.358 / sqrt(N) (alpha = 0.05); >= 100 samples required.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import ops
from ._lib import call


@dataclass
class Histogram:
    lo: float = 0.0
    hi: float = 0.0
    counts: list = field(default_factory=list)
    iter: int = 0
    layer: str = ""

    def total(self) -> int:
        return int(sum(self.counts))


def _host_histogram(x: np.ndarray, bins: int):
    x = np.asarray(x, dtype=np.float32).ravel()
    fin = x[np.isfinite(x)]
    m = float(np.float32(np.abs(fin).max())) if fin.size else 0.0
    lo, hi = (-m, m) if m > 0.0 else (-1.0, 1.0)
    idx = np.floor((fin.astype(np.float64) - lo) * (bins / (hi - lo))).astype(np.int64)
    idx = np.clip(idx, 0, bins - 1)
    return lo, hi, np.bincount(idx, minlength=bins).astype(np.int64)


def make_histogram(samples, bins: int = 64, iter: int = 0, layer: str = "") -> Histogram:
    """stats.hpp `make_histogram`: on the GPU for a CUDA tensor, else numpy."""
    if not 1 <= bins <= 8192:
        raise ValueError("make_histogram: bins must be in [1, 8192]")
    if isinstance(samples, torch.Tensor) and samples.is_cuda:
        x = samples.detach().contiguous().reshape(-1).float()
        counts = torch.empty(bins, dtype=torch.int64, device=x.device)
        lo_hi = torch.empty(2, dtype=torch.float64, device=x.device)
        call("i8t_histogram", ops.ctx(), ops._p(x), x.numel(), bins, ops._p(counts), ops._p(lo_hi))
        lh = lo_hi.cpu().tolist()
        return Histogram(lh[0], lh[1], counts.cpu().tolist(), iter, layer)
    if isinstance(samples, torch.Tensor):
        samples = samples.detach().numpy()
    lo, hi, counts = _host_histogram(samples, bins)
    return Histogram(lo, hi, counts.tolist(), iter, layer)


class DistFamily(Enum):
    GAUSSIAN = 0
    LAPLACE = 1
    STUDENT_T = 2


def family_name(f: DistFamily) -> str:
    return {DistFamily.GAUSSIAN: "Gaussian", DistFamily.LAPLACE: "Laplace", DistFamily.STUDENT_T: "StudentT"}[f]


@dataclass
class DistFit:
    family: DistFamily = DistFamily.GAUSSIAN
    location: float = 0.0
    scale: float = 1.0
    nu: float = 0.0
    ks: float = 0.0
    critical: float = 0.0

    def rejected(self) -> bool:
        return self.ks > self.critical


def gaussian_cdf(x: float, mu: float, sigma: float) -> float:
    return 0.5 * math.erfc(-(x - mu) / (sigma * math.sqrt(2.0)))


def laplace_cdf(x: float, mu: float, b: float) -> float:
    z = (x - mu) / b
    return 0.5 * math.exp(z) if z < 0.0 else 1.0 - 0.5 * math.exp(-z)


def _betacf(a: float, b: float, x: float) -> float:
    """Continued fraction of the regularised incomplete beta (modified Lentz)."""
    tiny = 1e-300
    qab, qap, qam = a + b, a + 1.0, a - 1.0
    c, d = 1.0, 1.0 - qab * x / qap
    d = 1.0 / (d if abs(d) > tiny else tiny)
    h = d
    for m in range(1, 400):
        m2 = 2 * m
        aa = m * (b - m) * x / ((qam + m2) * (a + m2))
        d = 1.0 + aa * d
        d = 1.0 / (d if abs(d) > tiny else tiny)
        c = 1.0 + aa / c
        c = c if abs(c) > tiny else tiny
        h *= d * c
        aa = -(a + m) * (qab + m) * x / ((a + m2) * (qap + m2))
        d = 1.0 + aa * d
        d = 1.0 / (d if abs(d) > tiny else tiny)
        c = 1.0 + aa / c
        c = c if abs(c) > tiny else tiny
        de = d * c
        h *= de
        if abs(de - 1.0) < 1e-16:
            break
    return h


def _betainc(a: float, b: float, x: float) -> float:
    if x <= 0.0:
        return 0.0
    if x >= 1.0:
        return 1.0
    lbt = math.lgamma(a + b) - math.lgamma(a) - math.lgamma(b) + a * math.log(x) + b * math.log1p(-x)
    if x < (a + 1.0) / (a + b + 2.0):
        return math.exp(lbt) * _betacf(a, b, x) / a
    return 1.0 - math.exp(lbt) * _betacf(b, a, 1.0 - x) / b


def student_t_cdf(x: float, mu: float, sigma: float, nu: float) -> float:
    t = (x - mu) / sigma
    tail = 0.5 * _betainc(0.5 * nu, 0.5, nu / (nu + t * t))
    return 1.0 - tail if t > 0.0 else tail


def dist_cdf(fit: DistFit, x: float) -> float:
    if fit.family == DistFamily.GAUSSIAN:
        return gaussian_cdf(x, fit.location, fit.scale)
    if fit.family == DistFamily.LAPLACE:
        return laplace_cdf(x, fit.location, fit.scale)
    return student_t_cdf(x, fit.location, fit.scale, fit.nu)


def _samples(samples) -> np.ndarray:
    if isinstance(samples, torch.Tensor):
        samples = samples.detach().float().cpu().numpy()
    x = np.asarray(samples, dtype=np.float32).ravel().astype(np.float64)
    if x.size == 0:
        raise ValueError("stats: empty sample set")
    return x


def _student_t_em(x: np.ndarray, nu: float, iters: int = 200):
    mu = float(np.median(x))
    s2 = float(np.mean((x - mu) ** 2)) or 1e-300
    for _ in range(iters):
        w = (nu + 1.0) / (nu + (x - mu) ** 2 / s2)
        mu_n = float(np.sum(w * x) / np.sum(w))
        s2_n = float(np.mean(w * (x - mu_n) ** 2))
        done = abs(mu_n - mu) <= 1e-14 * (abs(mu) + math.sqrt(s2)) and abs(s2_n - s2) <= 1e-12 * s2
        mu, s2 = mu_n, max(s2_n, 1e-300)
        if done:
            break
    sigma = math.sqrt(s2)
    n = x.size
    ll = (n * (math.lgamma((nu + 1) / 2) - math.lgamma(nu / 2) - 0.5 * math.log(nu * math.pi) - math.log(sigma))
          - (nu + 1) / 2 * float(np.sum(np.log1p((x - mu) ** 2 / (nu * s2)))))
    return mu, sigma, ll


def fit_mle(family: DistFamily, samples) -> DistFit:
    """Maximum-likelihood fit (stats.hpp `fit_mle`)."""
    x = _samples(samples)
    if family == DistFamily.GAUSSIAN:
        mu = float(np.mean(x))
        return DistFit(family, mu, float(np.sqrt(np.mean((x - mu) ** 2))))
    if family == DistFamily.LAPLACE:
        mu = float(np.median(x))
        return DistFit(family, mu, float(np.mean(np.abs(x - mu))))
    best = None
    for nu in range(1, 101):
        mu, sigma, ll = _student_t_em(x, float(nu))
        if best is None or ll > best[3]:
            best = (float(nu), mu, sigma, ll)
    return DistFit(family, best[1], best[2], best[0])


def ks_statistic(samples, fit: DistFit) -> float:
    """Sup distance between the empirical CDF and the fitted one (>= 100 samples;
    zero-variance input raises, as stats.hpp states)."""
    x = np.sort(_samples(samples))
    n = x.size
    if n < 100:
        raise ValueError("ks_statistic: needs at least 100 samples")
    if not (fit.scale > 0.0) or x[0] == x[-1]:
        raise ValueError("ks_statistic: degenerate (zero-variance) sample set")
    f = np.array([dist_cdf(fit, float(v)) for v in x])
    i = np.arange(1, n + 1, dtype=np.float64)
    return float(max(np.max(i / n - f), np.max(f - (i - 1) / n)))


def fit_and_test(family: DistFamily, samples) -> DistFit:
    x = _samples(samples)
    fit = fit_mle(family, x)
    fit.ks = ks_statistic(x, fit)
    fit.critical = 1.358 / math.sqrt(x.size)
    return fit


@dataclass
class SnapshotSummary:
    layer: str = ""
    iter: int = 0
    min: float = 0.0
    max: float = 0.0
    range: float = 0.0
    max_abs: float = 0.0
    kurtosis_proxy: float = 0.0


def summarize_samples(layer: str, iter: int, samples) -> SnapshotSummary:
    """min / max / range / max|x| / E[x^4] / E[x^2]^2 of a sample set."""
    x = _samples(samples)
    m2 = float(np.mean(x * x))
    m4 = float(np.mean(x ** 4))
    lo, hi = float(x.min()), float(x.max())
    return SnapshotSummary(layer, iter, lo, hi, hi - lo, max(abs(lo), abs(hi)), m4 / (m2 * m2) if m2 > 0.0 else 0.0)
