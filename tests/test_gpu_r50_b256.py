"""Parity at the benchmarked configuration: ResNet-50 layers at batch 256
(BASELINE.json configs[2]), one per conv code path the bench launches, with
the operand layouts, split counts and tile queues the model uses at b256.

* forward and backward-data: exact int32 accumulators and float outputs for
  images 0, 1 and N-1 (the first tile, a tile crossing an image boundary and
  the ragged tail) against the direct-loop oracle (oracle.c) on those images --
  each output image depends only on its own input image;
* backward-weight over the FULL batch (depth M = N*P*Q up to 3.2 M, far past
  the reference's 130000 bound): the int64 accumulator and the float gW of the
  model's direct mode (split partials rescaled without the int64 copy) exact
  against oracle/bigconv.py (exact float64-GEMM evaluation, pinned to oracle.c
  by tests/test_oracle_bigconv.py);
* the block-input quantiser i8t_bn_act_quant at b256 (BN statistics + apply +
  ReLU + nearest quantise in one pass) against the oracle BN followed by the
  oracle quantiser, with the +-1 decisions flipped by BN's last-bit statistics
  counted and bounded.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import bigconv as B
from oracle import lib as O

pytestmark = pytest.mark.gpu

CA, CW, CG = 3.3, 0.4, 2e-4
LAYERS = {  # name: (n, c, h, k, kernel, stride, pad) -- the path each one takes on the device
    "stem_7x7s2": (256, 3, 224, 64, 7, 2, 3),        # tap-folded narrow-channel gather; wgrad M = 3.2 M
    "l1_3x3": (256, 64, 56, 64, 3, 1, 1),            # shifted-window fwd / dgrad; 64-wide wgrad
    "l1_1x1_expand": (256, 64, 56, 256, 1, 1, 0),    # 1x1 TMA operands
    "l2_3x3s2": (256, 128, 56, 128, 3, 2, 1),        # strided gather fwd; four-phase dgrad
    "l2_downsample": (256, 256, 56, 512, 1, 2, 0),   # 1x1 stride 2; phase dgrad with zero phases
    "l3_3x3": (256, 256, 14, 256, 3, 1, 1),          # gathered (cp.async) 3x3 at 256 channels
    "l4_1x1": (256, 2048, 7, 512, 1, 1, 0),          # deep few-output wgrad: split-phase reducer
}


def _rnd(rng, shape, zero_frac):
    x = rng.integers(-127, 128, size=shape, dtype=np.int8)
    x[rng.random(shape, dtype=np.float32) < zero_frac] = 0
    return x


def _dev_nhwc(x_nhwc, c_pad):
    t = torch.zeros(x_nhwc.shape[:-1] + (c_pad,), dtype=torch.int8)
    t[..., :x_nhwc.shape[-1]] = torch.from_numpy(x_nhwc)
    return t.cuda()


@pytest.mark.parametrize("name", list(LAYERS))
def test_resnet50_b256_layer_exact(name, ops):
    n, c, h, k, kk, s, p = LAYERS[name]
    pg = ops.geom(n, c, h, h, k, kk, kk, s, p)
    og = O.geom(n, c, h, h, k, kk, kk, s, p)
    P, Q = O.out_hw(og)
    rng = np.random.default_rng(sum(name.encode()))
    a = _rnd(rng, (n, h, h, c), 0.5)             # NHWC, as on the device
    gz = _rnd(rng, (n, P, Q, k), 0.6)
    w = _rnd(rng, (k, c, kk, kk), 0.0)
    c_pad, k_pad = ops.pad4(c), ops.pad4(k)
    a_d, g_d = _dev_nhwc(a, c_pad), _dev_nhwc(gz, k_pad)
    w_d = torch.from_numpy(w).cuda()
    w_krsc, ld = ops.kcrs_to_krsc_i8(w_d, c_pad)
    w_crsk, ldt = ops.kcrs_to_crsk_i8(w_d, k_pad)
    z, acc = ops.conv_fwd_nhwc(pg, a_d, c_pad, w_krsc, ld, CA, CW, want_acc=True)
    z, acc = z.view(n, P, Q, k), acc.view(n, P, Q, k)
    sa, sw, sg = O.quant_scale(CA), O.quant_scale(CW), O.quant_scale(CG)
    imgs = [0, 1, n - 1]
    sub = O.geom(len(imgs), c, h, h, k, kk, kk, s, p)
    a_sub = np.ascontiguousarray(a[imgs].transpose(0, 3, 1, 2))
    acc_r, z_r = O.conv_fwd(a_sub, w, sub, sa, sw)
    np.testing.assert_array_equal(acc[imgs].permute(0, 3, 1, 2).cpu().numpy(), acc_r)
    np.testing.assert_array_equal(z[imgs].permute(0, 3, 1, 2).cpu().numpy(), z_r)
    if name != "stem_7x7s2":  # the model never runs the stem's backward-data (image gradient discarded)
        ga, dacc = ops.conv_dgrad_nhwc(pg, g_d, k_pad, w_crsk, ldt, CG, CW, want_acc=True)
        ga, dacc = ga.view(n, h, h, c), dacc.view(n, h, h, c)
        g_sub = np.ascontiguousarray(gz[imgs].transpose(0, 3, 1, 2))
        dacc_r, ga_r = O.conv_dgrad(g_sub, w, sub, sg, sw)
        np.testing.assert_array_equal(dacc[imgs].permute(0, 3, 1, 2).cpu().numpy().astype(np.int64), dacc_r)
        np.testing.assert_array_equal(ga[imgs].permute(0, 3, 1, 2).cpu().numpy(), ga_r)
    # backward-weight over the whole batch: int64 accumulator (data-parallel form) ...
    gw, wacc = ops.conv_wgrad_nhwc(pg, g_d, k_pad, a_d, c_pad, CG, CA, out_kcrs=True)
    wacc_r = B.wgrad_acc(gz, a, kk, kk, s, s, p, p)
    wacc = wacc.view(kk, kk, c_pad, k)[:, :, :c, :].permute(3, 2, 0, 1).cpu().numpy()
    np.testing.assert_array_equal(wacc, wacc_r)
    gw_r = B.rescale(wacc_r, sg, sa)
    np.testing.assert_array_equal(gw.cpu().numpy(), gw_r)
    # ... and the single-device direct mode the bench runs (no int64 copy)
    gw2 = torch.empty_like(gw)
    ops.call("i8t_conv_wgrad", ops.ctx(), C.byref(pg), g_d, k_pad, a_d, c_pad, ops._dev_f32(CG),
             ops._dev_f32(CA), None, gw2, 1)
    np.testing.assert_array_equal(gw2.cpu().numpy(), gw_r)


def test_bn_act_quant_b256_flips_bounded(ops):
    """i8t_bn_fwd_stats + i8t_bn_act_quant on a b256 56x56x64 layer against the
    oracle BatchNorm2d forward (layers.cpp:262-295) -> ReLU -> nearest quantise
    (quantize.cpp:16-31).  BN statistics are double sums in a different order,
    so a value at a rounding boundary may flip by one level."""
    n, h, c = 256, 56, 64
    m = n * h * h
    rng = np.random.default_rng(7)
    mu = rng.normal(0, 0.5, c).astype(np.float32)
    sd = rng.uniform(0.2, 3.0, c).astype(np.float32)
    z = (rng.standard_normal((n, h, h, c), dtype=np.float32) * sd + mu).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.normal(0, 0.2, c).astype(np.float32)
    clip = 2.7
    zd = torch.from_numpy(z).cuda()
    stats = torch.zeros(6 * c, dtype=torch.float64, device="cuda")
    rm, rv = torch.zeros(c, device="cuda"), torch.ones(c, device="cuda")
    ops.call("i8t_bn_fwd_stats", ops.ctx(), zd, m, c, C.c_double(0.1), C.c_double(1e-5), stats, rm, rv)
    q = torch.empty((n, h, h, c), dtype=torch.int8, device="cuda")
    amax = torch.zeros(1, device="cuda")
    ops.call("i8t_bn_act_quant", ops.ctx(), zd, m, c, stats, torch.from_numpy(gamma).cuda(),
             torch.from_numpy(beta).cuda(), 1, ops._dev_f32(clip), q, amax)
    # oracle: BN forward (train) in NCHW, ReLU, nearest quantiser
    x = np.ascontiguousarray(z.transpose(0, 3, 1, 2))
    y = np.empty_like(x)
    xhat = np.empty_like(x)
    invstd = np.empty(c, np.float64)
    rm_r, rv_r = np.zeros(c, np.float32), np.ones(c, np.float32)
    O.lib().or_bn_forward_train(x, n, c, h * h, gamma, beta, rm_r, rv_r, 0.1, 1e-5, y, xhat, invstd)
    y = np.where(y > 0, y, np.float32(0.0)).astype(np.float32)
    q_r, _ = O.quantize(y, clip)
    q_d = q.permute(0, 3, 1, 2).cpu().numpy()
    diff = q_d.astype(np.int32) - q_r
    flips = int(np.count_nonzero(diff))
    assert np.abs(diff).max() <= 1
    assert flips <= m * c // 1_000_000, flips      # <= 1 per million decisions
    np.testing.assert_allclose(rm.cpu().numpy(), rm_r, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(rv.cpu().numpy(), rv_r, rtol=1e-6, atol=1e-7)
    assert float(amax.item()) == float(O.max_abs(y))
    print(f"bn_act_quant b256: {flips} flips in {m * c} decisions")
