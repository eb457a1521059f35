"""GPU: I8FT v1 checkpoints interoperate with the reference's own
save_checkpoint / load_checkpoint (checkpoint.cpp:61-135, compiled unmodified
into oracle/_ref): a file the reference wrote after INT8 training loads into
the device trainer bit for bit (parameters, buffers, clip states, clip_w /
clip_a), written back unchanged it is byte-identical, and a file the device
trainer wrote after further steps loads into the reference.  The net is the
reference's tiny_cnn (models.cpp:22-40) rebuilt from this package's layers
with the same leaf names."""
import numpy as np
import pytest
import torch

from oracle import ref as R

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref absent")]


def _gpu_tiny_cnn():
    from paper_1912_12607_b200.layers import (AvgPool2d, BatchNorm2d, Conv2d, Dense, MaxPool2d, ReLU, Sequential,
                                              int8_replace)
    from paper_1912_12607_b200.models import Model
    from paper_1912_12607_b200.trainer import TrainConfig, Trainer
    net = Sequential()
    net.add("conv1", Conv2d(3, 4, 3, 1, 1))
    net.add("bn1", BatchNorm2d(4))
    net.add("relu1", ReLU())
    net.add("pool1", MaxPool2d(2, 2))
    net.add("conv2", Conv2d(4, 8, 3, 1, 1))
    net.add("bn2", BatchNorm2d(8))
    net.add("relu2", ReLU())
    net.add("pool2", MaxPool2d(2, 2))
    net.add("gap", AvgPool2d(8, 8))
    net.add("fc", Dense(8, 10))
    m = Model("tiny_cnn", net, 10, (3, 32, 32))
    int8_replace(net)
    return m, Trainer(m, TrainConfig(base_lr=0.05, clip_period=2, seed=3))


def _gpu_tensors(tr):
    from paper_1912_12607_b200.checkpoint import _tensors
    return {k: v.detach().cpu().numpy() for k, v in _tensors(tr).items()}


def test_checkpoint_v1_cross_read(tmp_path):
    from paper_1912_12607_b200.checkpoint import load_checkpoint, save_checkpoint
    from paper_1912_12607_b200.trainer import synthetic_batch
    rm = R.RefModel("tiny_cnn", seed=5, side=32, classes=10)
    nq = rm.int8_replace()
    rtr = R.RefTrainer(rm, base_lr=0.05, clip_period=2)
    rng = np.random.default_rng(0)
    for it in range(3):  # INT8 steps: clip states, clip_w / clip_a and BN running stats become non-trivial
        x = rng.standard_normal((8, 3, 32, 32)).astype(np.float32)
        y = rng.integers(0, 10, 8).astype(np.int32)
        assert not rtr.train_step(x, y, it, 10, nq)["diverged"]
    p1 = str(tmp_path / "ref.i8ft")
    rm.save(p1)
    m, tr = _gpu_tiny_cnn()
    assert load_checkpoint(tr, p1) == 0  # a bare v1 file: no resume sidecar
    tr.sync_states()
    ref_t, got = rm.tensors(), _gpu_tensors(tr)
    assert sorted(ref_t) == sorted(got)
    for k, v in ref_t.items():
        np.testing.assert_array_equal(got[k], v, err_msg=k)
    views = tr.arena.read_views()
    for i, ((path, layer), v) in enumerate(zip(tr.quant_layers, views)):
        f, cs = rtr.quant_state(i)
        assert (v.clip, v.last_dc, v.iter_of_last_update) == (cs.clip, cs.last_dc, cs.iter_of_last_update), path
        assert float(layer.qs.clip_w.item()) == f[0] and float(layer.qs.clip_a.item()) == f[1], path
    # written back unchanged: byte-identical to the reference's file
    p2 = str(tmp_path / "dev.i8ft")
    save_checkpoint(tr, p2, iteration=3, resume=False)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    # the device trains on; the reference loads what it writes
    x, y = synthetic_batch(m, 8, 1)
    for it in range(3, 5):
        assert not tr.train_step(x, y, it, 10).diverged
    p3 = str(tmp_path / "dev2.i8ft")
    save_checkpoint(tr, p3, iteration=5)
    rm2 = R.RefModel("tiny_cnn", seed=9, side=32, classes=10)
    rm2.load(p3)
    got = _gpu_tensors(tr)
    for k, v in rm2.tensors().items():
        np.testing.assert_array_equal(v, got[k], err_msg=k)
    # and the resume sidecar restores the stream exactly
    m2, tr2 = _gpu_tiny_cnn()
    assert load_checkpoint(tr2, p3) == 5
    assert int(tr2.grad_stream.item()) == int(tr.grad_stream.item())
    assert torch.equal(tr2.pflat, tr.pflat)
