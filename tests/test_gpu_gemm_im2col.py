"""GPU: gemm_i8_fused_lhs (gemm.cpp:49-64) and im2col_i8 / im2col_channel_i8
(conv.cpp:23-47, 98-106) on the device against the CPU oracle -- the
reference's fused == unfused contract incl. the LCG stream (test_kernels.cpp:
120-142), its im2col known layouts (:144-161), and ragged stochastic
quantisation (numel % 4 != 0) with exactly one draw per element."""
import numpy as np
import pytest
import torch

from oracle import lib as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,n", [(9, 40, 13), (7, 41, 5), (300, 1000, 200), (1, 3, 1)])
def test_gemm_fused_lhs_matches_unfused_oracle(ops, m, k, n):
    rng = np.random.default_rng(m * k + n)
    a = rng.standard_normal((m, k)).astype(np.float32)
    b = rng.integers(-127, 128, (k, n)).astype(np.int8)
    clip = float(O.max_abs(a))
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    # stochastic: draws in row-major order from the caller's stream
    q_r, s_r = O.quantize(a, clip, True, 555)
    ref = O.gemm_i8(q_r, b)
    st = ops.new_lcg_state(555)
    got = ops.gemm_i8_fused_lhs(ad, clip, True, st, bd)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)
    assert ops.lcg_value(st) == s_r
    # nearest
    qn, _ = O.quantize(a, clip)
    np.testing.assert_array_equal(ops.gemm_i8_fused_lhs(ad, clip, False, None, bd).cpu().numpy(), O.gemm_i8(qn, b))
    # and unfused on the device gives the same
    st2 = ops.new_lcg_state(555)
    qd = ops.quantize(ad, clip, True, st2)
    np.testing.assert_array_equal(ops.gemm_i8(qd, bd).cpu().numpy(), ref)
    assert ops.lcg_value(st2) == s_r


def test_gemm_fused_lhs_errors(ops):
    a = torch.zeros((2, 3), device="cuda")
    with pytest.raises(ValueError):
        ops.gemm_i8_fused_lhs(a, 1.0, False, None, torch.zeros((2, 2), dtype=torch.int8, device="cuda"))
    with pytest.raises(ValueError):
        ops.gemm_i8_fused_lhs(a, 1.0, True, None, torch.zeros((3, 2), dtype=torch.int8, device="cuda"))
    a[0, 1] = float("nan")
    ops.gemm_i8_fused_lhs(a, 1.0, False, None, torch.zeros((3, 2), dtype=torch.int8, device="cuda"))
    with pytest.raises(ArithmeticError):
        ops.check()


@pytest.mark.parametrize("n", [1, 5, 4097, 100003])
def test_stochastic_quantize_ragged_length(ops, n):
    x = O.gaussian((n,), n, 1.0)
    q_r, s_r = O.quantize(x, 2.5, True, 91)
    st = ops.new_lcg_state(91)
    q = ops.quantize(torch.from_numpy(x).cuda(), 2.5, True, st)
    np.testing.assert_array_equal(q.cpu().numpy(), q_r)
    assert ops.lcg_value(st) == s_r


def test_im2col_known_layouts(ops):
    x = torch.arange(1, 10, dtype=torch.int8).reshape(1, 1, 3, 3).cuda()
    col = ops.im2col_i8(x, ops.geom(1, 1, 3, 3, 1, 2, 2)).cpu().numpy()
    assert col.shape == (4, 4)
    assert list(col[:, 0]) == [1, 2, 4, 5]  # column 0 = top-left 2x2 patch
    col2 = ops.im2col_i8(x, ops.geom(1, 1, 3, 3, 1, 3, 3)).cpu().numpy()
    np.testing.assert_array_equal(col2.reshape(-1), np.arange(1, 10))


@pytest.mark.parametrize("geo", [(2, 3, 9, 9, 4, 3, 3, 2, 1, None, None), (1, 5, 7, 6, 2, 1, 7, 1, 0, 1, 3),
                                 (2, 4, 11, 10, 3, 7, 7, 2, 3, None, None), (3, 2, 5, 5, 1, 1, 1, 1, 0, None, None)])
def test_im2col_matches_oracle(ops, geo):
    n, c, h, w, k, kh, kw, s, p, sw, pw = geo
    og = O.geom(n, c, h, w, k, kh, kw, s, p, stride_w=sw, pad_w=pw)
    pg = ops.geom(n, c, h, w, k, kh, kw, s, p, stride_w=sw, pad_w=pw)
    x = np.random.default_rng(sum(geo[:8])).integers(-127, 128, (n, c, h, w)).astype(np.int8)
    ref = O.im2col_i8(x, og)
    xd = torch.from_numpy(x).cuda()
    np.testing.assert_array_equal(ops.im2col_i8(xd, pg).cpu().numpy(), ref)
    rows = kh * kw
    for ch in range(c):
        np.testing.assert_array_equal(ops.im2col_i8(xd, pg, ch).cpu().numpy(), ref[ch * rows:(ch + 1) * rows])
