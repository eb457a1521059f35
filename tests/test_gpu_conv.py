"""GPU parity: tcgen05 INT8 convolutions vs the CPU oracle (bit-exact int32 /
int64 accumulators and bit-exact float outputs given the same scales).

Geometries cover what the reference tests (conv == direct conv on random
small geometries incl. depthwise and stride 2, 1x1 identities, zero input,
test_kernels.cpp:163-300) plus the extensions the build needs: asymmetric
pad/stride (InceptionV3 1x7/7x1), floor-mode output, channels not a multiple
of 16 (vector widths 8 and 4), ResNet-50 / ResNet-20 layer shapes, and the
config-1 layer at full size.
"""
import numpy as np
import pytest
import torch

from oracle import lib as O

pytestmark = pytest.mark.gpu


def rnd_i8(rng, shape, zero_frac=0.0):
    x = rng.integers(-127, 128, size=shape).astype(np.int8)
    if zero_frac:
        x[rng.random(shape) < zero_frac] = 0
    return x


GEOMS = [
    # n, c, h, w, k, kh, kw, stride, pad, stride_w, pad_w, depthwise
    (1, 2, 5, 5, 3, 3, 3, 1, 1, None, None, False),      # spec's fixed case
    (2, 16, 8, 8, 16, 3, 3, 1, 1, None, None, False),
    (2, 64, 14, 14, 64, 3, 3, 1, 1, None, None, False),   # shifted-window path (conv_sw.cu)
    (2, 128, 28, 28, 128, 3, 3, 1, 1, None, None, False),  # shifted-window, two n-tiles
    (1, 64, 30, 30, 192, 3, 3, 1, 1, None, None, False),   # shifted-window, ragged tiles, K < BN
    (1, 64, 24, 24, 64, 1, 3, 1, 0, 1, 1, False),          # shifted-window 1x3
    (1, 64, 9, 9, 128, 3, 3, 2, 1, None, None, False),   # stride 2, floor mode
    (2, 32, 7, 7, 48, 1, 1, 1, 0, None, None, False),    # 1x1 (TMA-loaded operands)
    (3, 256, 9, 9, 512, 1, 1, 1, 0, None, None, False),  # 1x1, multi-tile M/N/K (TMA), ragged M
    (2, 144, 5, 7, 80, 1, 1, 1, 0, None, None, False),   # 1x1, K and C not tile multiples (TMA)
    (2, 48, 10, 10, 40, 1, 1, 2, 0, None, None, False),  # 1x1 stride 2 (downsample)
    (1, 3, 20, 20, 16, 7, 7, 2, 3, None, None, False),   # stem-like, C=3 (tap-folded)
    (2, 4, 12, 10, 24, 3, 5, 1, 1, 2, 2, False),         # C=4, kw=5, stride_w 2 (tap-folded)
    (2, 3, 30, 30, 64, 7, 7, 2, 3, None, None, False),   # stem, even size, K=64
    (2, 24, 9, 9, 24, 3, 3, 1, 1, None, None, False),    # C=24 (vec 8)
    (1, 32, 9, 11, 40, 1, 7, 1, 0, 1, 3, False),         # 1x7 asym pad
    (1, 32, 11, 9, 40, 7, 1, 1, 3, 1, 0, False),         # 7x1 asym pad
    (1, 256, 7, 7, 300, 3, 3, 1, 1, None, None, False),  # N > 256 tile
    (2, 192, 9, 9, 64, 3, 3, 2, 1, None, None, False),   # wgrad: 64-channel im2col halves straddling taps
    (1, 320, 7, 7, 32, 3, 3, 1, 1, None, None, False),   # wgrad: 64-channel halves, last half past M
    # strided dgrad through the stride-phase decomposition (k % 128 == 0)
    (2, 40, 11, 11, 128, 1, 1, 2, 0, None, None, False),  # 1x1 s2, zero phases, odd H
    (2, 64, 10, 10, 256, 3, 3, 2, 1, None, None, False),  # 3x3 s2, four phases
    (1, 24, 9, 10, 128, 3, 3, 2, 1, 1, 1, False),         # stride (2, 1)
    (1, 16, 13, 13, 128, 7, 7, 2, 3, None, None, False),  # 7x7 s2 p3
    # padded phase rows + 3-D TMA stores (9 <= Wq <= 32, H == 2 Hq)
    (1, 64, 18, 18, 128, 3, 3, 2, 1, None, None, False),  # Wq 9 -> 16-pixel rows, ragged last tile
    (3, 40, 20, 22, 128, 3, 3, 2, 1, None, None, False),  # Wq 11, C = 40 (clipped channel box)
    (2, 40, 60, 60, 128, 1, 1, 2, 0, None, None, False),  # 1x1 s2, Wq 30 -> 32-pixel rows
    (1, 24, 36, 20, 128, 3, 3, 2, 1, 1, 1, False),        # stride (2, 1): Wq 20, W stride C
    (2, 64, 14, 14, 128, 3, 3, 2, 1, None, None, False),  # Wq 7 -> 8-pixel rows, one ragged tile
    (1, 32, 12, 16, 128, 3, 3, 2, 1, None, None, False),  # Wq 8: no padding columns
    (3, 8, 6, 6, 8, 3, 3, 1, 1, None, None, True),       # depthwise
    (2, 40, 9, 9, 40, 3, 3, 2, 1, None, None, True),     # depthwise stride 2
    (4, 96, 28, 28, 96, 3, 3, 1, 1, None, None, True),   # depthwise, channel-quad kernels
    (3, 144, 29, 31, 144, 3, 3, 2, 1, None, None, True),  # depthwise stride 2, odd sizes
    (2, 6, 7, 7, 6, 3, 3, 1, 1, None, None, True),       # depthwise C % 4 != 0 (generic kernels)
]


def _geoms(g):
    n, c, h, w, k, kh, kw, s, p, sw, pw, dw = g
    return (O.geom(n, c, h, w, k, kh, kw, s, p, dw, True, sw, pw),
            __import__("paper_1912_12607_b200").ops.geom(n, c, h, w, k, kh, kw, s, p, dw, True, sw, pw))


@pytest.mark.parametrize("gi", range(len(GEOMS)))
def test_conv_fwd_dgrad_wgrad_match_oracle(gi, ops):
    og, pg = _geoms(GEOMS[gi])
    rng = np.random.default_rng(100 + gi)
    qa = rnd_i8(rng, (og.n, og.c, og.h, og.w), 0.3)
    qw = rnd_i8(rng, O.weight_shape(og))
    qg = rnd_i8(rng, O.output_shape(og), 0.5)
    ca, cw, cg = 1.27, 12.7, 3e-4
    sa, sw, sg = O.quant_scale(ca), O.quant_scale(cw), O.quant_scale(cg)
    acc_ref, z_ref = O.conv_fwd(qa, qw, og, sa, sw)
    dacc_ref, ga_ref = O.conv_dgrad(qg, qw, og, sg, sw)
    wacc_ref, gw_ref = O.conv_wgrad(qg, qa, og, sg, sa)

    t = lambda x: torch.from_numpy(x).cuda()
    z, acc = ops.conv2d_q(t(qa), ca, t(qw), cw, pg, want_acc=True)
    gw, ga, wacc, dacc = ops.conv2d_backward_q(t(qg), cg, t(qa), ca, t(qw), cw, pg, want_acc=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(acc.cpu().numpy(), acc_ref, err_msg="fwd int32 accumulator")
    np.testing.assert_array_equal(z.cpu().numpy(), z_ref, err_msg="fwd float output")
    np.testing.assert_array_equal(dacc.cpu().numpy().astype(np.int64), dacc_ref, err_msg="dgrad accumulator")
    np.testing.assert_array_equal(ga.cpu().numpy(), ga_ref, err_msg="dgrad float output")
    np.testing.assert_array_equal(wacc.cpu().numpy(), wacc_ref, err_msg="wgrad int64 accumulator")
    np.testing.assert_array_equal(gw.cpu().numpy(), gw_ref, err_msg="wgrad float output")


def test_gemm_i8_known_results(ops):
    a = torch.tensor([[1, 2], [3, 4]], dtype=torch.int8).cuda()
    b = torch.tensor([[5, 6], [7, 8]], dtype=torch.int8).cuda()
    assert ops.gemm_i8(a, b).cpu().tolist() == [[19, 22], [43, 50]]
    row = torch.full((1, 4), 127, dtype=torch.int8).cuda()
    col = torch.full((4, 1), 127, dtype=torch.int8).cuda()
    assert int(ops.gemm_i8(row, col).item()) == 64516


def test_gemm_i8_random_vs_oracle(ops):
    rng = np.random.default_rng(17)
    for _ in range(25):
        m, k, n = (int(v) for v in 1 + rng.integers(0, 16, 3))
        a, b = rnd_i8(rng, (m, k)), rnd_i8(rng, (k, n))
        got = ops.gemm_i8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
        np.testing.assert_array_equal(got, O.gemm_i8(a, b))
    a, b = rnd_i8(rng, (300, 1000)), rnd_i8(rng, (1000, 200))
    got = ops.gemm_i8(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    np.testing.assert_array_equal(got, O.gemm_i8(a, b))


def test_gemm_i8_depth_bound(ops):
    with pytest.raises(ValueError):
        ops.gemm_i8(torch.zeros((2, 3), dtype=torch.int8).cuda(), torch.zeros((2, 2), dtype=torch.int8).cuda())


def test_zero_gradient_and_zero_input(ops):
    og, pg = _geoms((1, 16, 6, 6, 16, 3, 3, 1, 1, None, None, False))
    z = torch.zeros((1, 16, 6, 6), dtype=torch.int8).cuda()
    w = torch.from_numpy(rnd_i8(np.random.default_rng(5), (16, 16, 3, 3))).cuda()
    out = ops.conv2d_q(z, 1.0, w, 1.0, pg)
    assert float(out.abs().max()) == 0.0
    gw, ga = ops.conv2d_backward_q(z, 1.0, z, 1.0, w, 1.0, pg)
    assert float(gw.abs().max()) == 0.0 and float(ga.abs().max()) == 0.0


def test_config1_full_size(ops):
    """Config 1 (N32 C=K=64 56x56 3x3 p1): forward and dgrad exact against the
    oracle; wgrad exact (int64); float outputs bit-exact."""
    og, pg = _geoms((32, 64, 56, 56, 64, 3, 3, 1, 1, None, None, False))
    rng = np.random.default_rng(1)
    qa = rnd_i8(rng, (32, 64, 56, 56), 0.5)
    qw = rnd_i8(rng, (64, 64, 3, 3))
    qg = rnd_i8(rng, (32, 64, 56, 56), 0.7)
    ca, cw, cg = 3.3, 0.4, 2e-4
    t = lambda x: torch.from_numpy(x).cuda()
    z = ops.conv2d_q(t(qa), ca, t(qw), cw, pg)
    gw, ga = ops.conv2d_backward_q(t(qg), cg, t(qa), ca, t(qw), cw, pg)
    _, z_ref = O.conv_fwd(qa, qw, og, O.quant_scale(ca), O.quant_scale(cw))
    np.testing.assert_array_equal(z.cpu().numpy(), z_ref)
    _, gw_ref = O.conv_wgrad(qg, qa, og, O.quant_scale(cg), O.quant_scale(ca))
    np.testing.assert_array_equal(gw.cpu().numpy(), gw_ref)
    _, ga_ref = O.conv_dgrad(qg, qw, og, O.quant_scale(cg), O.quant_scale(cw))
    np.testing.assert_array_equal(ga.cpu().numpy(), ga_ref)


@pytest.mark.parametrize("shape", [
    # ResNet-50 layer shapes at reduced batch (n, c, h, k, kh, stride, pad)
    (4, 256, 56, 64, 1, 1, 0),
    (4, 64, 56, 64, 3, 1, 1),
    (4, 128, 56, 128, 3, 2, 1),
    (4, 512, 28, 1024, 1, 2, 0),
    (2, 512, 7, 2048, 1, 1, 0),
])
def test_resnet50_layer_shapes(shape, ops):
    n, c, h, k, kh, s, p = shape
    og, pg = _geoms((n, c, h, h, k, kh, kh, s, p, None, None, False))
    rng = np.random.default_rng(sum(shape))
    qa = rnd_i8(rng, (n, c, h, h), 0.5)
    qw = rnd_i8(rng, (k, c, kh, kh))
    qg = rnd_i8(rng, O.output_shape(og), 0.6)
    t = lambda x: torch.from_numpy(x).cuda()
    z, acc = ops.conv2d_q(t(qa), 1.0, t(qw), 1.0, pg, want_acc=True)
    gw, ga, wacc, dacc = ops.conv2d_backward_q(t(qg), 1.0, t(qa), 1.0, t(qw), 1.0, pg, want_acc=True)
    acc_ref, _ = O.conv_fwd(qa, qw, og, 1.0, 1.0)
    np.testing.assert_array_equal(acc.cpu().numpy(), acc_ref)
    dacc_ref, _ = O.conv_dgrad(qg, qw, og, 1.0, 1.0)
    np.testing.assert_array_equal(dacc.cpu().numpy().astype(np.int64), dacc_ref)
    wacc_ref, _ = O.conv_wgrad(qg, qa, og, 1.0, 1.0)
    np.testing.assert_array_equal(wacc.cpu().numpy(), wacc_ref)


@pytest.mark.parametrize("shape", [(2, 40, 11, 128, 1, 2, 0), (2, 64, 10, 256, 3, 2, 1), (2, 64, 14, 64, 3, 1, 1),
                                   (2, 40, 36, 128, 1, 2, 0), (1, 64, 22, 256, 3, 2, 1)])
def test_dgrad_join_in_place_matches_dgrad_plus_add(shape, ops):
    """i8t_conv_dgrad_join with ga aliasing add_g (the projection-shortcut join
    accumulating into the main-branch gradient): equal to dgrad + add_g, the
    tap-less stride phases included (they are skipped, keeping add_g)."""
    import ctypes as C
    n, c, h, k, kk, s, p = shape
    g = ops.geom(n, c, h, h, k, kk, kk, s, p)
    P, Q = g.out_hw()
    cp, kp = ops.pad4(c), ops.pad4(k)
    gen = torch.Generator(device="cuda").manual_seed(7)
    qg = torch.randint(-127, 128, (n, P, Q, kp), dtype=torch.int8, device="cuda", generator=gen)
    w = torch.randn(k, c, kk, kk, device="cuda", generator=gen)
    _, qwt = ops.quantize_weight(w, float(w.abs().max()), c_pad=cp, k_pad=kp)
    cg = torch.tensor([0.02], device="cuda")
    cw = torch.tensor([float(w.abs().max())], device="cuda")
    add = torch.randn((n * h * h, c), device="cuda", generator=gen)
    add[add.abs() < 0.01] = 0.0  # +0 addends: -0 would stay -0 in place
    ref, _ = ops.conv_dgrad_nhwc(g, qg, kp, qwt, qwt.shape[1], cg, cw)
    ref = ref + add
    buf = add.clone()
    ops.call("i8t_conv_dgrad_join", ops.ctx(), C.byref(g), ops._p(qg), kp, ops._p(qwt), qwt.shape[1], ops._p(cg),
             ops._p(cw), ops._p(buf), ops._p(buf), None)
    torch.cuda.synchronize()
    assert torch.equal(buf.view(torch.int32), ref.view(torch.int32))
