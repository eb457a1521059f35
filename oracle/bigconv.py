"""Exact INT8 convolution accumulators at full batch size -- TEST
INFRASTRUCTURE ONLY (the checker of the b256 ResNet-50 layer tests; the
product never imports it).

The reference defines the backward-weight accumulator as the integer GEMM
GW[K x CRS] = Gmat[K x M] . col^T[M x CRS] (conv.cpp:186-195, M = N*P*Q) and
the forward one as Z = Wmat . col (conv.cpp:108-145).  oracle.c evaluates these
with direct integer loops, which at ResNet-50 batch 256 (M up to 3.2 M,
60 GOP for the stem's wgrad alone) takes minutes on the host.  Here the same
sums are evaluated by float64 GEMM, one filter tap at a time, over chunks of
M: every product (|q| <= 127) and every partial sum is an integer of
magnitude <= 127^2 * M < 2^53, so float64 represents each one exactly and the
result is the exact integer sum in any order -- identical to oracle.c's
int64 loops.  `exact_bound_ok` asserts the bound; tests/test_oracle_golden.py
pins these functions to oracle.c on random small geometries.

Layouts: activations / gradients NHWC int8 (the device layout), results KCRS
(wgrad, int64) or NHWC (forward, int64).  EXT geometry: separate stride / pad
per dimension, floor-mode output size.
"""
from __future__ import annotations

import numpy as np


def out_hw(h, w, kh, kw, sh, sw, ph, pw):
    return (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1


def exact_bound_ok(depth: int) -> bool:
    return 127 * 127 * depth < 2 ** 53


def _tap_view(xp, r, s, p, q, sh, sw):
    """[N, P, Q, C] view of the padded NHWC input under filter tap (r, s)."""
    return xp[:, r: r + sh * (p - 1) + 1: sh, s: s + sw * (q - 1) + 1: sw, :]


def wgrad_acc(g_nhwc: np.ndarray, a_nhwc: np.ndarray, kh, kw, sh=1, sw=1, ph=0, pw=0, chunk=1 << 17) -> np.ndarray:
    """int64 GW[K, C, kh, kw] = sum over (n, p, q) of g[n,p,q,k] * a[n, p*sh+r-ph, q*sw+s-pw, c]."""
    n, h, w, c = a_nhwc.shape
    p, q = out_hw(h, w, kh, kw, sh, sw, ph, pw)
    k = g_nhwc.shape[-1]
    assert g_nhwc.shape == (n, p, q, k)
    assert exact_bound_ok(n * p * q)
    xp = np.zeros((n, h + 2 * ph + sh, w + 2 * pw + sw, c), np.int8)
    xp[:, ph: ph + h, pw: pw + w, :] = a_nhwc
    out = np.zeros((k, c, kh, kw), np.float64)
    imgs = max(1, chunk // (p * q))
    for n0 in range(0, n, imgs):
        n1 = min(n, n0 + imgs)
        gm = g_nhwc[n0:n1].reshape(-1, k).astype(np.float64)          # [mc, K]
        for r in range(kh):
            for s in range(kw):
                am = _tap_view(xp[n0:n1], r, s, p, q, sh, sw).reshape(-1, c).astype(np.float64)  # [mc, C]
                out[:, :, r, s] += gm.T @ am
    return out.astype(np.int64)


def fwd_acc(a_nhwc: np.ndarray, w_kcrs: np.ndarray, sh=1, sw=1, ph=0, pw=0) -> np.ndarray:
    """int64 Z[N, P, Q, K] = sum over (c, r, s) of a[n, p*sh+r-ph, q*sw+s-pw, c] * w[k, c, r, s]."""
    n, h, w, c = a_nhwc.shape
    k, c2, kh, kw = w_kcrs.shape
    assert c2 == c and exact_bound_ok(c * kh * kw)
    p, q = out_hw(h, w, kh, kw, sh, sw, ph, pw)
    xp = np.zeros((n, h + 2 * ph + sh, w + 2 * pw + sw, c), np.int8)
    xp[:, ph: ph + h, pw: pw + w, :] = a_nhwc
    out = np.zeros((n * p * q, k), np.float64)
    wf = w_kcrs.astype(np.float64)
    for r in range(kh):
        for s in range(kw):
            am = _tap_view(xp, r, s, p, q, sh, sw).reshape(-1, c).astype(np.float64)
            out += am @ wf[:, :, r, s].T
    return out.astype(np.int64).reshape(n, p, q, k)


def rescale(acc: np.ndarray, s1: float, s2: float) -> np.ndarray:
    """float(double(s1) * double(s2) * double(acc)) (conv.cpp:140-143, 192-194)."""
    return ((np.float64(np.float32(s1)) * np.float64(np.float32(s2))) * acc.astype(np.float64)).astype(np.float32)
