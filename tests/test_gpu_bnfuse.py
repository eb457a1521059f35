"""GPU: fused BatchNorm2d + ReLU (csrc/bnfuse.cu) against a float64 numpy
restatement of the reference BN/ReLU/ResidualBlock (layers.cpp:230-344,
:451-456), and the fused quantiser entry points bit-exact against the
unfused kernel sequence they replace.

Tolerances: BN statistics are double sums reduced in a different order than
the reference's sequential loop -> mean/invstd rel 1e-12; every fp32 output
is a cast of a double expression of those statistics -> at most 1 ulp (the
comparison allows 2 ulp of the value's magnitude); grad_gamma/beta rel 1e-9.
The fused quantisers (bn_act_quant, quantize_gradient_bn) must equal
quantize_nearest_rows(bn_act(z)) / quantize_gradient(bn_bwd_apply(g, z))
bit-for-bit, including the LCG stream and the DSGC measurements."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref_bn(z, gamma, beta, momentum=0.1, eps=1e-5, rm=None, rv=None):
    """layers.cpp:262-290 on an NHWC [m, c] matrix (float64 arithmetic)."""
    zd = z.astype(np.float64)
    m = z.shape[0]
    mean = zd.sum(0) / m
    var = np.maximum((zd * zd).sum(0) / m - mean * mean, 0.0)
    inv = 1.0 / np.sqrt(var + eps)
    xv = (zd - mean) * inv
    y = (gamma.astype(np.float64) * xv + beta.astype(np.float64)).astype(np.float32)
    out = dict(mean=mean, inv=inv, xhat=xv.astype(np.float32), y=y)
    if rm is not None:
        out["rm"] = ((1.0 - momentum) * rm.astype(np.float64) + momentum * mean).astype(np.float32)
        out["rv"] = ((1.0 - momentum) * rv.astype(np.float64) + momentum * var).astype(np.float32)
    return out


def _ref_bn_bwd(g, ref, gamma):
    """layers.cpp:293-320."""
    m = g.shape[0]
    gd = g.astype(np.float64)
    xh = ref["xhat"].astype(np.float64)
    s1 = gd.sum(0)
    s2 = (gd * xh).sum(0)
    coeff = gamma.astype(np.float64) * ref["inv"]
    gi = (coeff * (gd - s1 / m - xh * s2 / m)).astype(np.float32)
    return gi, s1, s2


def _close(a, b, ulps=2):
    a, b = np.asarray(a, np.float32), np.asarray(b, np.float32)
    tol = ulps * np.spacing(np.maximum(np.abs(a), np.abs(b)).astype(np.float32))
    bad = np.abs(a.astype(np.float64) - b.astype(np.float64)) > tol
    assert not bad.any(), f"{bad.sum()} of {bad.size} differ; first {a[bad][:4]} vs {b[bad][:4]}"


def _data(m, c, seed):
    rng = np.random.default_rng(seed)
    z = (rng.standard_normal((m, c)) * rng.uniform(0.1, 3, c) + rng.uniform(-1, 1, c)).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.uniform(-0.3, 0.3, c).astype(np.float32)
    g = (rng.standard_normal((m, c)) * 1e-3).astype(np.float32)
    return z, gamma, beta, g


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _stats(ops, z, c, rm=None, rv=None):
    bn = torch.zeros(6 * c, dtype=torch.float64, device="cuda")
    ops.call("i8t_bn_fwd_stats", ops.ctx(), ops._p(z), z.numel() // c, c, C.c_double(0.1), C.c_double(1e-5),
             ops._p(bn), ops._p(rm), ops._p(rv))
    return bn


@pytest.mark.parametrize("m,c", [(6272, 64), (392, 256), (50, 12), (8, 2048), (1000, 132)])
def test_bn_forward_matches_reference(ops, m, c):
    z, gamma, beta, _ = _data(m, c, m + c)
    rm0 = np.linspace(-0.1, 0.1, c).astype(np.float32)
    rv0 = np.linspace(0.9, 1.1, c).astype(np.float32)
    ref = _ref_bn(z, gamma, beta, rm=rm0, rv=rv0)
    zt, gt, bt, rm, rv = t(z), t(gamma), t(beta), t(rm0), t(rv0)
    bn = _stats(ops, zt, c, rm, rv)
    b = bn.cpu().numpy()
    np.testing.assert_allclose(b[:c], ref["mean"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(b[c:2 * c], ref["inv"], rtol=1e-12)
    _close(rm.cpu().numpy(), ref["rm"])
    _close(rv.cpu().numpy(), ref["rv"])
    for relu in (0, 1):
        y = torch.empty_like(zt)
        ops.call("i8t_bn_act", ops.ctx(), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), relu, None, None,
                 None, None, None, ops._p(y))
        want = np.where(ref["y"] > 0, ref["y"], 0).astype(np.float32) if relu else ref["y"]
        _close(y.cpu().numpy(), want)


def test_bn_act_residual_forms(ops):
    m, c = 3136, 64
    z, gamma, beta, _ = _data(m, c, 1)
    z2, gamma2, beta2, _ = _data(m, c, 2)
    zt, gt, bt = t(z), t(gamma), t(beta)
    z2t, g2t, b2t = t(z2), t(gamma2), t(beta2)
    bn, bn2 = _stats(ops, zt, c), _stats(ops, z2t, c)
    y_main = torch.empty_like(zt)
    ops.call("i8t_bn_act", ops.ctx(), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), 0, None, None, None,
             None, None, ops._p(y_main))
    y_sc = torch.empty_like(zt)
    ops.call("i8t_bn_act", ops.ctx(), ops._p(z2t), m, c, ops._p(bn2), ops._p(g2t), ops._p(b2t), 0, None, None, None,
             None, None, ops._p(y_sc))
    want = torch.relu(y_main + y_sc)  # float add then ReLU (layers.cpp:451-456)
    for res_kind in ("dense", "lazy"):
        y = torch.empty_like(zt)
        if res_kind == "dense":
            args = (ops._p(y_sc), None, None, None, None)
        else:
            args = (None, ops._p(z2t), ops._p(bn2), ops._p(g2t), ops._p(b2t))
        ops.call("i8t_bn_act", ops.ctx(), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), 1, *args, ops._p(y))
        assert torch.equal(y, want)


@pytest.mark.parametrize("relu", [0, 1])
def test_bn_act_quant_equals_unfused(ops, relu):
    m, c = 12544, 64
    z, gamma, beta, _ = _data(m, c, 5 + relu)
    zt, gt, bt = t(z), t(gamma), t(beta)
    bn = _stats(ops, zt, c)
    y = torch.empty_like(zt)
    ops.call("i8t_bn_act", ops.ctx(), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), relu, None, None, None,
             None, None, ops._p(y))
    clip = torch.tensor([float(y.abs().max()) * 0.6], device="cuda")
    q_ref = torch.empty((m, c), dtype=torch.int8, device="cuda")
    amax_ref = torch.zeros(1, device="cuda")
    ops.call("i8t_quantize_nearest_rows", ops.ctx(), ops._p(y), m, c, ops._p(clip), ops._p(q_ref), c,
             ops._p(amax_ref), 1)
    q = torch.empty_like(q_ref)
    amax = torch.zeros(1, device="cuda")
    ops.call("i8t_bn_act_quant", ops.ctx(), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), relu,
             ops._p(clip), ops._p(q), ops._p(amax))
    assert torch.equal(q, q_ref)
    assert float(amax) == float(amax_ref) == float(y.abs().max())


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_bn_backward_matches_reference(ops, mode):
    m, c = 6272, 128
    z, gamma, beta, g = _data(m, c, 10 + mode)
    ref = _ref_bn(z, gamma, beta)
    mask_y = np.random.default_rng(3).standard_normal((m, c)).astype(np.float32)
    if mode == 1:
        gm = np.where(ref["y"] > 0, g, 0).astype(np.float32)
    elif mode == 2:
        gm = np.where(mask_y > 0, g, 0).astype(np.float32)
    else:
        gm = g
    gi_ref, s1, s2 = _ref_bn_bwd(gm, ref, gamma)
    zt, gt, bt, g_t, my = t(z), t(gamma), t(beta), t(g), t(mask_y)
    bn = _stats(ops, zt, c)
    gg, gb = torch.zeros(c, device="cuda"), torch.zeros(c, device="cuda")
    ops.call("i8t_bn_bwd_reduce", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), mode,
             ops._p(my) if mode == 2 else None, ops._p(gg), ops._p(gb))
    np.testing.assert_allclose(gb.cpu().numpy(), s1.astype(np.float32), rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(gg.cpu().numpy(), s2.astype(np.float32), rtol=1e-6, atol=1e-12)
    b = bn.cpu().numpy()
    # sums of +-terms: relative error is bounded against the largest sum, not each one
    k = gamma.astype(np.float64) * ref["inv"]  # bn[4c..5c) = gamma*invstd, bn[2c..4c) = k*s1/m, k*s2/m
    np.testing.assert_allclose(b[4 * c:5 * c], k, rtol=1e-9)
    np.testing.assert_allclose(b[2 * c:3 * c], k * s1 / m, rtol=1e-9, atol=1e-9 * np.abs(k * s1 / m).max())
    np.testing.assert_allclose(b[3 * c:4 * c], k * s2 / m, rtol=1e-9, atol=1e-9 * np.abs(k * s2 / m).max())
    gi = torch.empty_like(zt)
    ops.call("i8t_bn_bwd_apply", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), mode,
             ops._p(my) if mode == 2 else None, ops._p(gi))
    # cancellation in g - s1/m - xhat*s2/m: compare at the gradient's scale
    np.testing.assert_allclose(gi.cpu().numpy(), gi_ref, rtol=1e-6, atol=1e-7 * float(np.abs(gi_ref).max()))


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_quantize_gradient_bn_equals_unfused(ops, mode):
    n, hw, c = 8, 14 * 14, 64
    m = n * hw
    z, gamma, beta, g = _data(m, c, 20 + mode)
    mask_y = np.random.default_rng(4).standard_normal((m, c)).astype(np.float32)
    zt, gt, bt, g_t, my = t(z), t(gamma), t(beta), t(g), t(mask_y)
    bn = _stats(ops, zt, c)
    gg, gb = torch.zeros(c, device="cuda"), torch.zeros(c, device="cuda")
    myp = ops._p(my) if mode == 2 else None
    ops.call("i8t_bn_bwd_reduce", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), mode,
             myp, ops._p(gg), ops._p(gb))
    gi = torch.empty_like(zt)
    ops.call("i8t_bn_bwd_apply", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), mode,
             myp, ops._p(gi))
    gi4 = gi.view(n, 14, 14, c)
    # two states searched identically at iteration 0, then one non-due iteration each way
    sa, sb = ops.DsgcState(period=4), ops.DsgcState(period=4)
    la, lb = ops.new_lcg_state(77), ops.new_lcg_state(77)
    ops.quantize_gradient(sa, gi4, 0, la, nhwc=True)
    ops.quantize_gradient(sb, gi4, 0, lb, nhwc=True)
    sa.sync(), sb.sync()
    assert not sa.due(1) and not sb.due(1)
    q_ref = ops.quantize_gradient(sa, gi4, 1, la, nhwc=True)
    q = torch.empty_like(q_ref)
    ops.call("i8t_quantize_gradient_bn", ops.ctx(), sb.ptr, ops._p(g_t), ops._p(zt), n, c, hw, ops._p(bn), ops._p(gt),
             ops._p(bt), mode, myp, 1, C.c_double(20.0), C.c_double(0.1), ops.FORMS["exp"], ops._p(lb), ops._p(q))
    assert torch.equal(q, q_ref)
    assert ops.lcg_value(la) == ops.lcg_value(lb)
    va, vb = sa.view(), sb.view()
    for f in ("clip", "scale", "max_abs", "last_dc", "lr_scale", "eps_norm", "ghat_sqnorm", "iter_of_last_update"):
        assert getattr(va, f) == getattr(vb, f), f


def test_add_masked(ops):
    rng = np.random.default_rng(9)
    a, g, y = (rng.standard_normal(4096).astype(np.float32) for _ in range(3))
    out = torch.empty(4096, device="cuda")
    ops.call("i8t_add_masked", ops.ctx(), ops._p(t(a)), ops._p(t(g)), ops._p(t(y)), 4096, ops._p(out))
    np.testing.assert_array_equal(out.cpu().numpy(), a + np.where(y > 0, g, 0).astype(np.float32))


def _pack_bits(mask):
    """bool [n] -> int32 words, bit e%32 of word e/32 (the i8t_bn_act_q layout)."""
    flat = np.asarray(mask, bool).reshape(-1)
    pad = (-flat.size) % 32
    words = np.packbits(np.concatenate([flat, np.zeros(pad, bool)]).reshape(-1, 32)[:, ::-1], axis=1)
    return np.ascontiguousarray(words).view(">u4").astype(np.uint32).view(np.int32).reshape(-1)


def test_packed_mask_mode3_equals_mode2(ops):
    """mask mode 3 (packed bits of y > 0, written by i8t_bn_act_q) gives the same
    BN backward, fused gradient quantiser and residual join as mode 2 on y."""
    m, c = 3136, 64
    z, gamma, beta, g = _data(m, c, 21)
    z2, g2, b2, _ = _data(m, c, 22)
    zt, gt, bt, g_t = t(z), t(gamma), t(beta), t(g)
    bn, bn2 = _stats(ops, zt, c), _stats(ops, t(z2), c)
    # the block output y = relu(bn(z) + bn2(z2)) and its packed mask from the same pass
    y = torch.empty_like(zt)
    bits = torch.zeros(((m * c + 31) // 32,), dtype=torch.int32, device="cuda")
    ops.call("i8t_bn_act_q", ops.ctx(), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), 1, None, ops._p(t(z2)),
             ops._p(bn2), ops._p(t(g2)), ops._p(t(b2)), ops._p(y), None, None, None, ops._p(bits))
    assert np.array_equal(bits.cpu().numpy(), _pack_bits(y.cpu().numpy() > 0))
    outs = {}
    for mode, mk in ((2, y), (3, bits)):
        bnm = bn.clone()
        gg, gb = torch.zeros(c, device="cuda"), torch.zeros(c, device="cuda")
        ops.call("i8t_bn_bwd_reduce", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bnm), ops._p(gt), ops._p(bt),
                 mode, ops._p(mk), ops._p(gg), ops._p(gb))
        gi = torch.empty_like(zt)
        ops.call("i8t_bn_bwd_apply", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bnm), ops._p(gt), ops._p(bt),
                 mode, ops._p(mk), ops._p(gi))
        outs[mode] = (gg.clone(), gb.clone(), bnm.clone(), gi.clone())
    for x2, x3 in zip(outs[2], outs[3]):
        assert torch.equal(x2, x3)
    a = torch.randn(m * c, device="cuda")
    o2, o3 = torch.empty_like(a), torch.empty_like(a)
    ops.call("i8t_add_masked", ops.ctx(), ops._p(a), ops._p(g_t), ops._p(y), m * c, ops._p(o2))
    ops.call("i8t_add_masked_bits", ops.ctx(), ops._p(a), ops._p(g_t), ops._p(bits), m * c, ops._p(o3))
    assert torch.equal(o2, o3)


@pytest.mark.parametrize("m,c", [(3136, 64), (1000, 256), (49 * 8, 2048)])
def test_bn_bwd_reduce_join_equals_join_then_reduce(ops, m, c):
    """i8t_bn_bwd_reduce_join (identity-shortcut join materialised inside the
    BN backward column sums) == i8t_add_masked_bits then i8t_bn_bwd_reduce with
    mask mode 3: the joined gradient, grad_gamma / grad_beta and the BN
    coefficients bit for bit."""
    z, gamma, beta, g = _data(m, c, 31)
    rng = np.random.default_rng(32)
    zt, gt, bt, g_t = t(z), t(gamma), t(beta), t(g)
    a = t(rng.standard_normal((m, c)).astype(np.float32))
    jbits = t(_pack_bits(rng.random(m * c) < 0.6))
    mbits = t(_pack_bits(rng.random(m * c) < 0.5))
    bn = _stats(ops, zt, c)
    ref_g = torch.empty_like(zt)
    ops.call("i8t_add_masked_bits", ops.ctx(), ops._p(a), ops._p(g_t), ops._p(jbits), m * c, ops._p(ref_g))
    bn_r, bn_f = bn.clone(), bn.clone()
    gg_r, gb_r = torch.zeros(c, device="cuda"), torch.zeros(c, device="cuda")
    ops.call("i8t_bn_bwd_reduce", ops.ctx(), ops._p(ref_g), ops._p(zt), m, c, ops._p(bn_r), ops._p(gt), ops._p(bt), 3,
             ops._p(mbits), ops._p(gg_r), ops._p(gb_r))
    out = torch.empty_like(zt)
    gg_f, gb_f = torch.zeros(c, device="cuda"), torch.zeros(c, device="cuda")
    ops.call("i8t_bn_bwd_reduce_join", ops.ctx(), ops._p(a), ops._p(g_t), ops._p(jbits), ops._p(zt), m, c,
             ops._p(bn_f), ops._p(gt), ops._p(bt), ops._p(mbits), ops._p(gg_f), ops._p(gb_f), ops._p(out))
    assert torch.equal(out.view(torch.int32), ref_g.view(torch.int32))
    assert torch.equal(gg_f, gg_r) and torch.equal(gb_f, gb_r) and torch.equal(bn_f, bn_r)


def test_bn_rejects_bad_shapes(ops):
    z = torch.zeros(10, 6, device="cuda")
    bn = torch.zeros(30, dtype=torch.float64, device="cuda")
    with pytest.raises(ops.I8tError, match="c % 4"):  # I8T_EUNSUPPORTED: outside the kernels' envelope
        ops.call("i8t_bn_fwd_stats", ops.ctx(), z, 10, 6, C.c_double(0.1), C.c_double(1e-5), bn, None, None)


def _train(impl, name="resnet20", batch=16, steps=3, mode=None, join=True):
    from paper_1912_12607_b200 import layers as L
    from paper_1912_12607_b200.models import build_model
    from paper_1912_12607_b200.trainer import TrainConfig, Trainer, synthetic_batch
    old, old_join, old_proj = L.BN_IMPL, L.JOIN_FUSION, L.JOIN_PROJ
    L.BN_IMPL, L.JOIN_FUSION, L.JOIN_PROJ = impl, join, join
    try:
        m = build_model(name, seed=3)
        L.int8_replace(m.net)
        cfg = TrainConfig(base_lr=0.02, clip_period=2, seed=11)
        if mode is not None:
            cfg.mode = mode
        tr = Trainer(m, cfg)
        x, y = synthetic_batch(m, batch, 5)
        return tr, [tr.train_step(x, y, it, 100) for it in range(steps)]
    finally:
        L.BN_IMPL, L.JOIN_FUSION, L.JOIN_PROJ = old, old_join, old_proj


@pytest.mark.parametrize("name,batch", [("resnet20", 16), ("resnet50", 2), ("mobilenet_v2", 4), ("inception_v3", 2)])
def test_fused_equals_eager_bit_exact(name, batch):
    """Lazy BN/ReLU values (fused into the quantisers, residual adds and
    masks) give bit-identical training to materialising every value with the
    same kernels: losses, DSGC measurements, parameters and the LCG stream.
    Steps 0-3 with period 2 cover search and non-search iterations."""
    ta, ra = _train("fused", name, batch, 4)
    tb, rb = _train("eager", name, batch, 4)
    for a, b in zip(ra, rb):
        assert a.loss == b.loss
        for la, lb in zip(a.layers, b.layers):
            assert (la.clip, la.dc, la.eps_norm, la.ghat_sqnorm) == (lb.clip, lb.dc, lb.eps_norm, lb.ghat_sqnorm)
    assert torch.equal(ta.pflat, tb.pflat)
    assert int(ta.grad_stream.item()) == int(tb.grad_stream.item())


@pytest.mark.parametrize("name,batch", [("resnet20", 16), ("resnet50", 2)])
def test_residual_join_in_dgrad_epilogue_bit_exact(name, batch):
    """i8t_conv_dgrad_join (residual joins inside the dgrad epilogue, incl. the
    strided stride-phase path) trains bit-identically to dgrad + separate joins."""
    ta, ra = _train("fused", name, batch, 3, join=True)
    tb, rb = _train("fused", name, batch, 3, join=False)
    for a, b in zip(ra, rb):
        assert a.loss == b.loss
    assert torch.equal(ta.pflat, tb.pflat)
    assert int(ta.grad_stream.item()) == int(tb.grad_stream.item())


def test_fused_bn_tracks_torch_bn_fp32_mode():
    """FP32 mode (no quantisers): double-arithmetic BN vs torch's fp32 BN on
    ResNet-20 agree to fp32 rounding.  (Deeper nets at tiny batch amplify the
    rounding until ReLU masks flip -- tools/bn_diag.py -- so the bit-exact
    fused-vs-eager test above carries the plumbing check.)"""
    from paper_1912_12607_b200.layers import Mode
    tf32 = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False  # TF32 input rounding would amplify 1-ulp BN differences
    try:
        ta, ra = _train("fused", "resnet20", 16, 2, Mode.FP32)
        tb, rb = _train("torch", "resnet20", 16, 2, Mode.FP32)
    finally:
        torch.backends.cudnn.allow_tf32 = tf32
    for a, b in zip(ra, rb):
        assert a.loss == pytest.approx(b.loss, rel=1e-5)
    torch.testing.assert_close(ta.pflat, tb.pflat, rtol=1e-4, atol=1e-6)


def test_fused_int8_tracks_torch_bn():
    """INT8 ResNet-20: BN rounding differences flip a few quantiser decisions
    per layer; training stays finite and close to the torch-BN run."""
    _, ra = _train("fused", "resnet20", 16)
    _, rb = _train("torch", "resnet20", 16)
    assert ra[0].loss == pytest.approx(rb[0].loss, rel=3e-3)
    for a, b in zip(ra, rb):
        assert np.isfinite(a.loss) and not a.diverged
        assert a.loss == pytest.approx(b.loss, rel=2e-2)



@pytest.mark.parametrize("shape", [(2, 112, 112, 64, 3, 2, 1), (2, 15, 13, 32, 3, 2, 1), (3, 17, 15, 8, 3, 2, 0),
                                   (2, 9, 9, 12, 2, 2, 1), (1, 18, 22, 8, 3, 2, 1)])
@pytest.mark.parametrize("with_bn", [False, True])
def test_maxpool_matches_torch(ops, shape, with_bn):
    """csrc/pool.cu vs torch max_pool2d (+ its backward) on act(bn(z)) / x."""
    n, h, w, c, k, s, p = shape
    rng = np.random.default_rng(n * h + c)
    x = rng.standard_normal((n * h * w, c)).astype(np.float32)
    x[rng.random(x.shape) < 0.05] = 0.0  # ties
    xt = t(x)
    if with_bn:
        gamma, beta = t(rng.uniform(0.5, 1.5, c).astype(np.float32)), t(rng.uniform(-.3, .3, c).astype(np.float32))
        bn = _stats(ops, xt, c)
        act = torch.empty_like(xt)
        ops.call("i8t_bn_act", ops.ctx(), ops._p(xt), n * h * w, c, ops._p(bn), ops._p(gamma), ops._p(beta), 1, None,
                 None, None, None, None, ops._p(act))
    else:
        act = xt
    ref_in = act.view(n, h, w, c).permute(0, 3, 1, 2).contiguous().requires_grad_(True)
    ref = torch.nn.functional.max_pool2d(ref_in, k, s, p)
    P, Q = ref.shape[2], ref.shape[3]
    y = torch.empty((n, P, Q, c), device="cuda")
    idx = torch.empty((n, P, Q, c), dtype=torch.uint8, device="cuda")
    ops.call("i8t_maxpool_fwd", ops.ctx(), ops._p(xt), n, h, w, c, k, s, p, ops._p(bn) if with_bn else None,
             ops._p(gamma) if with_bn else None, ops._p(beta) if with_bn else None, 1 if with_bn else 0, ops._p(y),
             ops._p(idx))
    assert torch.equal(y, ref.detach().permute(0, 2, 3, 1))
    gy = torch.randn((n, P, Q, c), device="cuda")
    ref.backward(gy.permute(0, 3, 1, 2))
    gx = torch.empty((n, h, w, c), device="cuda")
    ops.call("i8t_maxpool_bwd", ops.ctx(), ops._p(gy), ops._p(idx), n, h, w, c, k, s, p, ops._p(gx))
    torch.testing.assert_close(gx, ref_in.grad.permute(0, 2, 3, 1), rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("case", ["collide", "negative_gamma", "all_clamped", "nan"])
def test_maxpool_bn_first_max_slot_exact(ops, case):
    """The BN-fused max pool finds the window maximum from the raw extreme z
    (act(bn(.)) is monotone per channel); its one-byte slot must still be the
    reference's FIRST maximum of act(bn(z)) in window order (Pool2d's `>`,
    layers.cpp:366-373) -- checked against a brute-force first-max over the
    materialised act(bn(z)) on inputs built to collide after rounding: values
    one ulp apart squeezed by a small BN slope, negative gammas (decreasing
    map), all-clamped windows, NaN inputs."""
    n, h, w, c, k, s, p = 2, 24, 20, 64, 3, 2, 1
    rng = np.random.default_rng(["collide", "negative_gamma", "all_clamped", "nan"].index(case))
    x = rng.standard_normal((n * h * w, c)).astype(np.float32)
    gamma = rng.uniform(0.5, 1.5, c).astype(np.float32)
    beta = rng.uniform(-.3, .3, c).astype(np.float32)
    if case == "collide":  # a few distinct floats around 100 (one to three ulps apart), wide spread elsewhere
        base = np.float32(100.0)
        x[:, : c // 2] = base + (rng.integers(0, 4, (n * h * w, c // 2)) * np.spacing(base)).astype(np.float32)
        x[rng.random(x.shape) < 0.3] *= np.float32(50.0)
        gamma[: c // 2] = 1e-3
    elif case == "negative_gamma":
        gamma[::2] *= -1.0
        x[rng.random(x.shape) < 0.2] = 0.0
    elif case == "all_clamped":
        beta[:] = -40.0
    else:
        x[rng.random(x.shape) < 0.1] = np.nan
    xt = t(x)
    bn = _stats(ops, t(np.nan_to_num(x)), c)  # statistics from finite data
    gt, bt = t(gamma), t(beta)
    act = torch.empty_like(xt)
    ops.call("i8t_bn_act", ops.ctx(), ops._p(xt), n * h * w, c, ops._p(bn), ops._p(gt), ops._p(bt), 1, None, None, None,
             None, None, ops._p(act))
    P, Q = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
    y = torch.empty((n, P, Q, c), device="cuda")
    idx = torch.empty((n, P, Q, c), dtype=torch.uint8, device="cuda")
    ops.call("i8t_maxpool_fwd", ops.ctx(), ops._p(xt), n, h, w, c, k, s, p, ops._p(bn), ops._p(gt), ops._p(bt), 1,
             ops._p(y), ops._p(idx))
    a = act.view(n, h, w, c).cpu().numpy()
    want_y = np.empty((n, P, Q, c), np.float32)
    want_i = np.empty((n, P, Q, c), np.uint8)
    for pp in range(P):
        for qq in range(Q):
            best = np.full((n, c), -np.inf, np.float32)
            arg = np.zeros((n, c), np.uint8)
            for dy in range(k):
                for dx in range(k):
                    hh, ww = pp * s - p + dy, qq * s - p + dx
                    if not (0 <= hh < h and 0 <= ww < w):
                        continue
                    v = a[:, hh, ww, :]
                    upd = v > best
                    best = np.where(upd, v, best)
                    arg = np.where(upd, dy * k + dx, arg)
            want_y[:, pp, qq, :], want_i[:, pp, qq, :] = best, arg
    np.testing.assert_array_equal(y.cpu().numpy(), want_y)
    np.testing.assert_array_equal(idx.cpu().numpy(), want_i)


def test_global_avgpool_matches_reference_order(ops):
    """i8t_global_avgpool_fwd / _bwd (Pool2d kAvg over the whole map,
    layers.cpp:383-414): the window summed in double in the reference's
    sequential order then float(acc / hw); backward g / float(hw) everywhere."""
    rng = np.random.default_rng(51)
    n, h, w, c = 4, 7, 7, 96
    x = rng.standard_normal((n, h, w, c)).astype(np.float32) * np.float32(3.0)
    y = torch.empty((n, c), device="cuda")
    ops.call("i8t_global_avgpool_fwd", ops.ctx(), ops._p(t(x)), n, h * w, c, ops._p(y))
    acc = np.zeros((n, c), np.float64)
    for k in range(h * w):  # reference order: row-major over the window
        acc += x.reshape(n, h * w, c)[:, k, :].astype(np.float64)
    np.testing.assert_array_equal(y.cpu().numpy(), (acc / (h * w)).astype(np.float32))
    g = rng.standard_normal((n, c)).astype(np.float32)
    gx = torch.empty((n, h, w, c), device="cuda")
    ops.call("i8t_global_avgpool_bwd", ops.ctx(), ops._p(t(g)), n, h * w, c, ops._p(gx))
    ref = np.broadcast_to((g / np.float32(h * w))[:, None, None, :], (n, h, w, c))
    np.testing.assert_array_equal(gx.cpu().numpy(), ref)


def test_bn_bwd_apply_stats_feeds_the_search(ops):
    """i8t_bn_bwd_apply_stats writes the same gz as i8t_bn_bwd_apply plus the
    DSGC search's first-pass statistics (max|g|, non-finite, sum g^2), and a
    due i8t_quantize_gradient_stats search on them picks the clip the plain
    search picks."""
    n, hw, c = 8, 14 * 14, 64
    m = n * hw
    z, gamma, beta, g = _data(m, c, 71)
    zt, gt, bt, g_t = t(z), t(gamma), t(beta), t(g)
    bn = _stats(ops, zt, c)
    gg, gb = torch.zeros(c, device="cuda"), torch.zeros(c, device="cuda")
    ops.call("i8t_bn_bwd_reduce", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), 1,
             None, ops._p(gg), ops._p(gb))
    ref = torch.empty_like(zt)
    ops.call("i8t_bn_bwd_apply", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt), 1,
             None, ops._p(ref))
    out = torch.empty_like(zt)
    st3 = torch.zeros(3, dtype=torch.float64, device="cuda")
    ops.call("i8t_bn_bwd_apply_stats", ops.ctx(), ops._p(g_t), ops._p(zt), m, c, ops._p(bn), ops._p(gt), ops._p(bt),
             1, None, ops._p(out), ops._p(st3))
    assert torch.equal(out, ref)
    s = st3.cpu().numpy()
    o = out.cpu().numpy().astype(np.float64)
    assert s[0] == np.abs(o).max() and s[1] == 0.0
    assert s[2] == pytest.approx((o * o).sum(), rel=1e-12)
    g4 = out.view(n, 14, 14, c)
    sa, sb = ops.DsgcState(period=4), ops.DsgcState(period=4)
    la, lb = ops.new_lcg_state(5), ops.new_lcg_state(5)
    qa = ops.quantize_gradient(sa, g4, 0, la, nhwc=True)
    qb = torch.empty_like(qa)
    ops.call("i8t_quantize_gradient_stats", ops.ctx(), sb.ptr, ops._p(g4), n, c, hw, 0, 32, 2, 1, 1, 1,
             C.c_double(20.0), C.c_double(0.1), ops.FORMS["exp"], ops._p(lb), ops._p(qb), c, ops._p(st3))
    va, vb = sa.view(), sb.view()
    assert va.clip == vb.clip and torch.equal(qa, qb)
    assert vb.last_dc == pytest.approx(va.last_dc, abs=1e-12)


@pytest.mark.parametrize("m,c", [(3136, 64), (49 * 8, 2048)])
def test_bn_bwd_reduce_join2_equals_two_reductions(ops, m, c):
    """i8t_bn_bwd_reduce_join2 (the projection block's two BNs reduced on the
    same joined, masked gradient in one pass) == i8t_bn_bwd_reduce_join for the
    first BN and i8t_bn_bwd_reduce for the second, bit for bit."""
    z, gamma, beta, g = _data(m, c, 91)
    z2, gamma2, beta2, _ = _data(m, c, 92)
    rng = np.random.default_rng(93)
    zt, gt, bt, g_t, z2t, g2t, b2t = t(z), t(gamma), t(beta), t(g), t(z2), t(gamma2), t(beta2)
    a = t(rng.standard_normal((m, c)).astype(np.float32))
    jbits = t(_pack_bits(rng.random(m * c) < 0.6))
    mbits = t(_pack_bits(rng.random(m * c) < 0.5))
    bn, bn2 = _stats(ops, zt, c), _stats(ops, z2t, c)
    out_r = torch.empty_like(zt)
    bn_r, bn2_r = bn.clone(), bn2.clone()
    gg_r, gb_r, gg2_r, gb2_r = (torch.zeros(c, device="cuda") for _ in range(4))
    ops.call("i8t_bn_bwd_reduce_join", ops.ctx(), ops._p(a), ops._p(g_t), ops._p(jbits), ops._p(zt), m, c,
             ops._p(bn_r), ops._p(gt), ops._p(bt), ops._p(mbits), ops._p(gg_r), ops._p(gb_r), ops._p(out_r))
    ops.call("i8t_bn_bwd_reduce", ops.ctx(), ops._p(out_r), ops._p(z2t), m, c, ops._p(bn2_r), ops._p(g2t), ops._p(b2t),
             3, ops._p(mbits), ops._p(gg2_r), ops._p(gb2_r))
    out = torch.empty_like(zt)
    bn_f, bn2_f = bn.clone(), bn2.clone()
    gg_f, gb_f, gg2_f, gb2_f = (torch.zeros(c, device="cuda") for _ in range(4))
    ops.call("i8t_bn_bwd_reduce_join2", ops.ctx(), ops._p(a), ops._p(g_t), ops._p(jbits), ops._p(zt), m, c,
             ops._p(bn_f), ops._p(gt), ops._p(bt), ops._p(mbits), ops._p(gg_f), ops._p(gb_f), ops._p(z2t),
             ops._p(bn2_f), ops._p(g2t), ops._p(gg2_f), ops._p(gb2_f), ops._p(out))
    assert torch.equal(out.view(torch.int32), out_r.view(torch.int32))
    for x, y in ((gg_f, gg_r), (gb_f, gb_r), (bn_f, bn_r), (gg2_f, gg2_r), (gb2_f, gb2_r), (bn2_f, bn2_r)):
        assert torch.equal(x, y)
