"""GPU: the layer API and the per-step trainer.

* One INT8 Conv2d layer step through layers.py reproduces the reference's
  Conv2d::forward/backward (golden dump of layers.cpp:98-126 incl.
  quantize_gradient :19-59): z, gA, gW bit-exact, stream state exact,
  d_c / phi / eps / g_hat^2 within tolerance.
* Dense (fc) forward/backward against the oracle (1x1 conv + bias).
* ResNet-20 (config 2 shape) trains several steps: finite loss, the device LCG
  stream advances by exactly the number of draws the reference would take
  (sum of g_z sizes of all INT8 layers with a non-zero gradient), phi in
  [beta, 1], weights updated.
"""
import os

import numpy as np
import pytest
import torch

from oracle import lib as O

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def nhwc(a):
    return torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 3, 1))).cuda()


@pytest.mark.parametrize("li", range(2))
def test_conv_layer_step_matches_reference_golden(li):
    from paper_1912_12607_b200 import ops
    from paper_1912_12607_b200.layers import BackwardCtx, Conv2d, ForwardCtx, Mode, StateArena

    n, c, h, w, k, kh, kw, s, p, dw = (int(v) for v in G[f"layer{li}_g"])
    conv = Conv2d(c, k, kh, s, p)
    conv.set_quantized(True)
    conv.weight = torch.from_numpy(G[f"layer{li}_W"]).cuda()
    conv.grad_weight = torch.zeros_like(conv.weight)
    arena = StateArena()
    arena.register(conv)
    arena.build(100)
    z = conv.forward(nhwc(G[f"layer{li}_X"]), ForwardCtx(Mode.INT8, True, True))
    lcg = ops.new_lcg_state(int(G[f"layer{li}_stream"][0]))
    ga = conv.backward(nhwc(G[f"layer{li}_GO"]), BackwardCtx(Mode.INT8, 0, lcg))
    ops.check()
    np.testing.assert_array_equal(z.permute(0, 3, 1, 2).cpu().numpy(), G[f"layer{li}_z"])
    np.testing.assert_array_equal(ga.permute(0, 3, 1, 2).cpu().numpy(), G[f"layer{li}_ga"])
    np.testing.assert_array_equal(conv.grad_weight.cpu().numpy(), G[f"layer{li}_gw"])
    assert ops.lcg_value(lcg) == int(G[f"layer{li}_stream"][1])
    v = arena.read_views()[0]
    st = G[f"layer{li}_stats"]
    assert np.float32(conv.qs.clip_w.item()) == np.float32(st[0])
    assert np.float32(conv.qs.clip_a.item()) == np.float32(st[1])
    assert np.float32(v.clip) == np.float32(st[2])
    assert v.last_dc == pytest.approx(st[3], abs=1e-9)
    assert v.lr_scale == pytest.approx(st[4], rel=1e-8)
    assert v.eps_norm == pytest.approx(st[5], rel=1e-9)
    assert v.ghat_sqnorm == pytest.approx(st[6], rel=1e-9)


def test_dense_layer_matches_oracle():
    from paper_1912_12607_b200 import ops
    from paper_1912_12607_b200.layers import BackwardCtx, Dense, ForwardCtx, Mode, StateArena

    n, fin, fout = 32, 64, 10
    fc = Dense(fin, fout)
    fc.set_quantized(True)
    W = O.gaussian((fout, fin, 1, 1), 9, 0.1)
    fc.conv.weight = torch.from_numpy(W).cuda()
    fc.conv.grad_weight = torch.zeros_like(fc.conv.weight)
    fc.bias = torch.linspace(-0.1, 0.1, fout).cuda()
    arena = StateArena()
    arena.register(fc)
    arena.build(100)
    X = O.gaussian((n, fin), 10, 1.0, True)
    GO = O.gradient_like((n, fout), 11, 1e-3, 0.0)
    z = fc.forward(torch.from_numpy(X).cuda(), ForwardCtx())
    lcg = ops.new_lcg_state(5)
    gi = fc.backward(torch.from_numpy(GO).cuda(), BackwardCtx(Mode.INT8, 0, lcg))
    ops.check()
    g = O.geom(n, fin, 1, 1, fout, 1, 1)
    cw, ca = O.max_abs(W), O.max_abs(X)
    qw, _ = O.quantize(W, cw)
    qa, _ = O.quantize(X.reshape(n, fin, 1, 1), ca)
    _, zr = O.conv_fwd(qa, qw, g, O.quant_scale(ca), O.quant_scale(cw))
    zr = zr.reshape(n, fout) + fc.bias.cpu().numpy()
    np.testing.assert_array_equal(z.cpu().numpy(), zr)
    st = O.new_clip_state(100)
    qg, sg, stream, _ = O.quantize_gradient(st, GO.reshape(n, fout, 1, 1), 0, 5)
    _, gir = O.conv_dgrad(qg, qw, g, sg, O.quant_scale(cw))
    _, gwr = O.conv_wgrad(qg, qa, g, sg, O.quant_scale(ca))
    np.testing.assert_array_equal(gi.cpu().numpy(), gir.reshape(n, fin))
    np.testing.assert_array_equal(fc.conv.grad_weight.cpu().numpy(), gwr)
    gb = (qg.reshape(n, fout).astype(np.int64).sum(0) * np.float64(sg)).astype(np.float32)
    np.testing.assert_array_equal(fc.grad_bias.cpu().numpy(), gb)
    assert ops.lcg_value(lcg) == stream


def test_resnet20_trains_with_exact_stream_accounting():
    from paper_1912_12607_b200 import ops
    from paper_1912_12607_b200.layers import int8_replace
    from paper_1912_12607_b200.models import build_model
    from paper_1912_12607_b200.trainer import TrainConfig, Trainer, synthetic_batch

    model = build_model("resnet20", seed=3)
    assert int8_replace(model.net) == 22  # 19 convs + 2 shortcut 1x1 + fc
    tr = Trainer(model, TrainConfig(base_lr=0.05, clip_period=2, seed=7))
    x, y = synthetic_batch(model, 32, 1)
    w0 = model.net.children[0][1].weight.clone()
    state = 7
    for it in range(4):
        rep = tr.train_step(x, y, it, 100)
        assert not rep.diverged and np.isfinite(rep.loss)
        for path, layer in tr.quant_layers:  # no zero-gradient skips in this run
            assert layer.qs.dsgc.view().flags & 2 == 0, path
        for ls in rep.layers:
            assert 0.1 <= ls.lr_scale <= 1.0 and ls.clip > 0 and ls.eps_norm > 0
    assert not torch.equal(w0, model.net.children[0][1].weight)
    # stream accounting: rerun one step and compare the advance with the sum of gradient sizes
    before = ops.lcg_value(tr.grad_stream)
    sizes = []
    orig = type(model.net.children[0][1]).backward

    def spy(self, gz, ctx):
        sizes.append(gz.numel())
        return orig(self, gz, ctx)
    type(model.net.children[0][1]).backward = spy
    try:
        tr.train_step(x, y, 4, 100)
    finally:
        type(model.net.children[0][1]).backward = orig
    after = ops.lcg_value(tr.grad_stream)
    assert len(sizes) == 22
    assert after == O.lcg_jump(before, sum(sizes))


def test_softmax_ce_device_matches_reference_formula():
    """i8t_softmax_ce (SoftmaxCrossEntropy::loss_and_grad, layers.cpp:507-529):
    loss and g_logits against a float64 numpy restatement, plus the divergence
    flag on a non-finite logit."""
    import numpy as np
    import torch
    from paper_1912_12607_b200.layers import SoftmaxCrossEntropy
    rng = np.random.default_rng(61)
    n, k = 37, 1000
    x = (rng.standard_normal((n, k)) * 4).astype(np.float32)
    lab = rng.integers(0, k, n)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    loss, g = SoftmaxCrossEntropy.loss_and_grad(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda(), 2 * n,
                                                bad=bad)
    xd = x.astype(np.float64)
    mx = xd.max(1, keepdims=True)
    logz = mx + np.log(np.exp(xd - mx).sum(1, keepdims=True))
    ref_loss = float((logz[:, 0] - xd[np.arange(n), lab]).sum() / (2 * n))
    p = np.exp(xd - logz)
    p[np.arange(n), lab] -= 1.0
    ref_g = (p / (2 * n)).astype(np.float32)
    assert float(loss) == pytest.approx(ref_loss, rel=1e-13)
    np.testing.assert_allclose(g.cpu().numpy(), ref_g, rtol=2e-7, atol=1e-12)
    assert int(bad) == 0
    x[3, 17] = np.inf
    SoftmaxCrossEntropy.loss_and_grad(torch.from_numpy(x).cuda(), torch.from_numpy(lab).cuda(), n, bad=bad)
    assert int(bad) == 1


def test_side_stream_weight_gradients_bit_identical():
    """Weight gradients on the side stream (trainer.WGRAD_STREAM) train
    bit-identically to the in-line weight gradients: parameters, losses, DSGC
    measurements and the LCG stream after three ResNet-20 steps (one a search
    step)."""
    import torch
    from paper_1912_12607_b200 import trainer as T
    from paper_1912_12607_b200.models import build_model
    from paper_1912_12607_b200.layers import int8_replace

    def run(flag):
        old = T.WGRAD_STREAM
        T.WGRAD_STREAM = flag
        try:
            torch.manual_seed(0)
            m = build_model("resnet20", num_classes=10)
            int8_replace(m.net)
            tr = T.Trainer(m, T.TrainConfig(base_lr=0.05, clip_period=2, seed=3))
            x, y = T.synthetic_batch(m, 16, 5)
            reps = [tr.train_step(x, y, it, 10) for it in range(3)]
            return tr, reps
        finally:
            T.WGRAD_STREAM = old

    ta, ra = run(True)
    tb, rb = run(False)
    for a, b in zip(ra, rb):
        assert a.loss == b.loss
        for la, lb in zip(a.layers, b.layers):
            assert (la.clip, la.dc) == (lb.clip, lb.dc)
    assert torch.equal(ta.pflat, tb.pflat)
    assert int(ta.grad_stream.item()) == int(tb.grad_stream.item())
