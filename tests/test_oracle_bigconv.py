"""Pins oracle/bigconv.py (exact float64-GEMM evaluation of the INT8 conv
accumulators, used to check full-batch ResNet-50 layers) to the direct-loop
oracle (oracle.c, itself pinned to the compiled reference) on random
geometries incl. stride 2, asymmetric padding, 7x7 and ragged sizes.  CPU only."""
import numpy as np
import pytest

from oracle import bigconv as B
from oracle import lib as O

GEOMS = [  # n, c, h, w, k, kh, kw, sh, sw, ph, pw
    (2, 3, 17, 15, 8, 7, 7, 2, 2, 3, 3),
    (3, 16, 9, 9, 12, 3, 3, 1, 1, 1, 1),
    (2, 8, 11, 10, 16, 3, 3, 2, 2, 1, 1),
    (1, 32, 7, 7, 20, 1, 1, 1, 1, 0, 0),
    (2, 12, 9, 9, 24, 1, 1, 2, 2, 0, 0),
    (1, 6, 9, 11, 5, 1, 7, 1, 1, 0, 3),
]


@pytest.mark.parametrize("geo", GEOMS)
def test_bigconv_matches_direct_oracle(geo):
    n, c, h, w, k, kh, kw, sh, sw, ph, pw = geo
    rng = np.random.default_rng(sum(geo))
    g = O.geom(n, c, h, w, k, kh, kw, sh, ph, stride_w=sw, pad_w=pw)
    p, q = O.out_hw(g)
    a = rng.integers(-127, 128, (n, c, h, w)).astype(np.int8)
    wt = rng.integers(-127, 128, (k, c, kh, kw)).astype(np.int8)
    gz = rng.integers(-127, 128, (n, k, p, q)).astype(np.int8)
    a_n, g_n = a.transpose(0, 2, 3, 1).copy(), gz.transpose(0, 2, 3, 1).copy()
    acc_f, z_f = O.conv_fwd(a, wt, g, 0.031, 0.0042)
    mine = B.fwd_acc(a_n, wt, sh, sw, ph, pw)
    np.testing.assert_array_equal(mine.transpose(0, 3, 1, 2), acc_f)
    np.testing.assert_array_equal(B.rescale(mine, 0.031, 0.0042).transpose(0, 3, 1, 2), z_f)
    acc_w, gw = O.conv_wgrad(gz, a, g, 2e-5, 0.031)
    mine_w = B.wgrad_acc(g_n, a_n, kh, kw, sh, sw, ph, pw, chunk=37)  # several M chunks
    np.testing.assert_array_equal(mine_w, acc_w)
    np.testing.assert_array_equal(B.rescale(mine_w, 2e-5, 0.031), gw)


def test_bigconv_exactness_bound():
    assert B.exact_bound_ok(3_211_264)          # the ResNet-50 stem wgrad depth at batch 256
    assert not B.exact_bound_ok(2 ** 53 // 127 ** 2 + 1)
