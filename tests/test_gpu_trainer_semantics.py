"""GPU: Trainer::train_step semantics against the step-level oracle
(oracle/model.py, pinned to the compiled reference Trainer):

* calibrate + finish_calibration / refresh_wa_clips (train.cpp:29-46): the
  FP32 forward's activation maxima per layer (fp32 convolutions, no TF32)
  and the clips they become; clip_w = max_abs(W) exactly;
* the divergence return (train.cpp:73-77): non-finite logits -> diverged
  before backward, no LCG draws, no update, no DSGC state change;
* the bad-gradient return (train.cpp:87-95): a non-finite parameter gradient
  -> diverged, parameters untouched (the device flag gates the SGD launch),
  while the backward's draws and DSGC updates stand as in the reference;
* SGD with momentum (train.cpp:104-111): buf = float(m*buf + g) and
  w -= float(lr*buf) track the oracle (first step: identical inputs, so the
  buffers equal the gradients up to BN's last-bit statistics).
"""
import math

import numpy as np
import pytest
import torch

from oracle import model as M

pytestmark = pytest.mark.gpu


def _pair(batch=32, **cfg):
    from test_gpu_step_parity import _oracle_from
    from paper_1912_12607_b200.layers import int8_replace
    from paper_1912_12607_b200.models import build_model
    from paper_1912_12607_b200.trainer import TrainConfig, Trainer, synthetic_batch
    m = build_model("resnet20", seed=4)
    int8_replace(m.net)
    tr = Trainer(m, TrainConfig(base_lr=0.05, clip_period=2, seed=11, **cfg))
    net, otr = _oracle_from(tr)
    if cfg:
        otr = M.Trainer(net, M.TrainConfig(base_lr=0.05, clip_period=2, seed=11, **cfg))
    x, y = synthetic_batch(m, batch, 1)
    return m, tr, net, otr, x, y


def _nchw(t):
    return t.permute(0, 3, 1, 2).contiguous().cpu().numpy()


def test_calibrate_and_refresh_clips_match_oracle():
    m, tr, net, otr, x, y = _pair()
    tr.calibrate(x)
    otr.calibrate(_nchw(x))
    for (path, gl), (_, ol) in zip(tr.quant_layers, otr.quant_layers):
        assert float(gl.qs.pending_amax.item()) == pytest.approx(float(ol.qs.pending_amax), rel=1e-5), path
    tr.finish_calibration()
    otr.finish_calibration()
    for (path, gl), (_, ol) in zip(tr.quant_layers, otr.quant_layers):
        assert float(gl.qs.clip_w.item()) == float(ol.qs.clip_w), path  # max_abs(W): exact
        assert float(gl.qs.clip_a.item()) == pytest.approx(float(ol.qs.clip_a), rel=1e-5), path
        assert float(gl.qs.pending_amax.item()) == 0.0 and gl.qs.clip_w_set and gl.qs.clip_a_set
        # the clips differ by <= 1e-6 relative (fp32 conv rounding).  That is enough
        # to move the freshly initialised INT8 net's loss by ~1 % (every clip
        # shifts every quantiser boundary), so the oracle adopts the device's clips
        # and the INT8 step on them must then agree to double rounding
        ol.qs.clip_a = np.float32(gl.qs.clip_a.item())
    rep = tr.train_step(x, y, 0, 10)
    orep = otr.train_step(_nchw(x), y.cpu().numpy().astype(np.int32), 0, 10)
    assert rep.loss == pytest.approx(orep["loss"], rel=1e-12)


def test_divergence_return_matches_oracle():
    m, tr, net, otr, x, y = _pair()
    fc = tr.leaves[-1][1]
    fc.bias[3] = float("inf")
    M.named_tensors(net)["fc.bias"][3] = np.inf
    before = tr.pflat.clone()
    s0 = int(tr.grad_stream.item())
    rep = tr.train_step(x, y, 0, 10)
    orep = otr.train_step(_nchw(x), y.cpu().numpy().astype(np.int32), 0, 10)
    assert rep.diverged and orep["diverged"]
    assert math.isnan(rep.loss) or math.isinf(rep.loss)
    assert int(tr.grad_stream.item()) == s0 and otr.stream[0] == 11  # no draws
    assert torch.equal(torch.nan_to_num(tr.pflat), torch.nan_to_num(before))
    tr.sync_states()
    assert all(v.iter_of_last_update < 0 for v in tr.arena.read_views())


def test_bad_gradient_skips_update():
    from paper_1912_12607_b200 import layers as L
    m, tr, net, otr, x, y = _pair()
    rep0 = tr.train_step(x, y, 0, 10)  # a clean step first
    before = tr.pflat.clone()
    s_before = int(tr.grad_stream.item())
    target = tr.quant_layers[5][1]

    def poison(conv, ev, **t):  # a non-finite weight gradient, as a huge update would produce
        if ev == "bwd" and conv is target:
            conv.grad_weight.view(-1)[7] = float("nan")
    L.TRACE = poison
    try:
        rep = tr.train_step(x, y, 1, 10)
    finally:
        L.TRACE = None
    assert not rep0.diverged and rep.diverged
    assert torch.equal(tr.pflat, before)                 # update skipped (train.cpp:87-95)
    assert int(tr.grad_stream.item()) != s_before         # the backward's draws were consumed
    assert all(ls.dc >= 0 for ls in rep.layers)           # DSGC statistics of the backward stand
    rep2 = tr.train_step(x, y, 2, 10)                      # and training continues
    assert not rep2.diverged and not torch.equal(tr.pflat, before)


def test_momentum_step_matches_oracle():
    """Teacher-forced on gradients: after each step the oracle adopts the
    device's parameters; momentum buffers must agree exactly."""
    from test_gpu_step_parity import _adopt
    m, tr, net, otr, x, y = _pair(momentum=0.9)
    assert tr.mflat is not None
    for it in range(3):
        rep = tr.train_step(x, y, it, 10)
        orep = otr.train_step(_nchw(x), y.cpu().numpy().astype(np.int32), it, 10)
        assert rep.loss == pytest.approx(orep["loss"], rel=1e-9 if it == 0 else 2e-3)
        if it == 0:  # identical inputs: the buffers are the gradients (BN's last bits aside)
            segs = [p for _, layer in tr.leaves for p in layer.params()]
            om = [otr.mom[(i, j)] for i, (_, l) in enumerate(otr.leaves) for j in range(len(l.params()))]
            mf = tr.mflat.cpu().numpy()
            for p, ob in zip(segs, om):  # a parameter's momentum sits at its offset in the parameter arena
                off = (p.value.data_ptr() - tr.pflat.data_ptr()) // 4
                got = mf[off:off + p.value.numel()].reshape(ob.shape)
                np.testing.assert_allclose(got, ob, rtol=1e-4, atol=1e-6 * float(np.abs(ob).max()), err_msg=p.name)
        _adopt(tr, net)
