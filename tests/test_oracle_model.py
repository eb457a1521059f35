"""Pins the step-level oracle (oracle/model.py) against the compiled, unmodified
reference Trainer (oracle/_ref, train.cpp:12-120 on models.cpp / layers.cpp
nets): identical parameters, losses, per-layer DSGC / DCLR statistics and
QuantStates after several INT8 steps -- bit for bit -- including the
calibration pass, search and non-search iterations, momentum, the
clip-search-disabled mode and the divergence / bad-gradient returns.
CPU only (runs here; skipped where the reference build is absent)."""
import math

import numpy as np
import pytest

from oracle import lib as O
from oracle import model as M
from oracle import ref as R

pytestmark = pytest.mark.skipif(not R.available(), reason="reference build (oracle/_ref) absent")

SIDE = {"tiny_cnn": 32, "res_s1": 12, "mbv2_s1": 12}


def _pair(name, seed=5, **cfg):
    side = SIDE[name]
    rm = R.RefModel(name, seed=seed, side=side, classes=10)
    om = M.build(name, classes=10, side=side)
    rt, ot = rm.tensors(), M.named_tensors(om)
    assert sorted(rt) == sorted(ot)
    for k, v in rt.items():
        assert ot[k].shape == v.shape, k
        ot[k][...] = v
    assert rm.int8_replace() == M.int8_replace(om)
    rtr = R.RefTrainer(rm, **cfg)
    mcfg = {k: v for k, v in cfg.items() if k not in ("lr_scaling", "clip_enabled")}
    mcfg.update(lr_scaling_enabled=cfg.get("lr_scaling", True), clip_enabled=cfg.get("clip_enabled", True))
    otr = M.Trainer(om, M.TrainConfig(**mcfg))
    return rm, om, rtr, otr, side


def _batch(side, n, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, 3, side, side)).astype(np.float32), rng.integers(0, 10, n).astype(np.int32)


def _same_state(rm, om, rtr, otr):
    rt, ot = rm.tensors(), M.named_tensors(om)
    for k in rt:
        np.testing.assert_array_equal(rt[k], ot[k], err_msg=k)
    for i, (_, l) in enumerate(otr.quant_layers):
        f, cs = rtr.quant_state(i)
        assert f[0] == l.qs.clip_w and f[1] == l.qs.clip_a and f[2] == l.qs.pending_amax
        assert cs.clip == l.qs.cs.clip and cs.last_dc == l.qs.cs.last_dc
        assert cs.iter_of_last_update == l.qs.cs.iter_of_last_update


def _run(name, steps=4, calibrate=True, n=8, **cfg):
    rm, om, rtr, otr, side = _pair(name, **cfg)
    if calibrate:
        x, _ = _batch(side, n, 99)
        rtr.calibrate(x)
        otr.calibrate(x)
        rtr.finish_calibration()
        otr.finish_calibration()
        _same_state(rm, om, rtr, otr)
    nq = len(otr.quant_layers)
    for it in range(steps):
        x, y = _batch(side, n, it)
        r = rtr.train_step(x, y, it, 50, nq)
        o = otr.train_step(x, y, it, 50)
        assert r["diverged"] == o["diverged"]
        assert r["loss"] == o["loss"] and r["base_lr_t"] == o["base_lr_t"]
        got = np.array([row[1:] for row in o["layers"]], np.float64)
        np.testing.assert_array_equal(r["layers"], got)
        _same_state(rm, om, rtr, otr)
    assert otr.stream[0] != cfg.get("seed", 1)  # the gradient stream was consumed
    return rm, om, rtr, otr


@pytest.mark.parametrize("name", ["tiny_cnn", "res_s1", "mbv2_s1"])
def test_trainer_steps_match_reference(name):
    _run(name, steps=5, clip_period=2)


def test_trainer_momentum_matches_reference():
    _run("res_s1", steps=4, momentum=0.9, clip_period=3)


def test_trainer_clip_search_disabled_constant_lr():
    _run("tiny_cnn", steps=3, clip_enabled=False, schedule="constant", lr_scaling=False)


def test_trainer_without_calibration_lazy_clips():
    _run("res_s1", steps=3, calibrate=False, clip_period=100)


def test_trainer_linear_form_grid_only():
    _run("mbv2_s1", steps=3, form="linear", rounds=0, grid=16, clip_period=2)


def test_divergence_return():
    rm, om, rtr, otr, side = _pair("tiny_cnn")
    nq = len(otr.quant_layers)
    x, y = _batch(side, 4, 1)
    # non-finite logits (an infinite fc bias): diverged before backward (train.cpp:73-77)
    bias = np.zeros(10, np.float32)
    bias[3] = np.inf
    rm.set_tensors({"fc.bias": bias})
    M.named_tensors(om)["fc.bias"][...] = bias
    r = rtr.train_step(x, y, 0, 10, nq)
    o = otr.train_step(x, y, 0, 10)
    assert r["diverged"] and o["diverged"]
    assert (math.isnan(r["loss"]) and math.isnan(o["loss"])) or r["loss"] == o["loss"]
    _same_state(rm, om, rtr, otr)
    assert otr.stream[0] == 1  # no draws consumed


def test_softmax_ce_and_pools_match_reference_layers():
    """The FP32 pieces alone: a tiny_cnn forward in FP32 inference mode (BN
    eval, max / avg Pool2d, FP32 conv and Dense) tracks identical activation
    maxima in both (calibrate), and softmax-CE is exact on extreme logits."""
    rm, om, rtr, otr, side = _pair("tiny_cnn")
    x, _ = _batch(side, 3, 7)
    rtr.calibrate(x * 100)
    otr.calibrate(x * 100)
    _same_state(rm, om, rtr, otr)
    logits = np.array([[1e4, -1e4, 0.0], [0.0, 0.0, 0.0], [-3.5, 88.0, 88.0]], np.float32)
    loss, g = M.softmax_ce(logits, np.array([0, 2, 1], np.int32))
    assert math.isfinite(loss) and g.dtype == np.float32
    np.testing.assert_allclose(g.sum(1), 0.0, atol=1e-7)
