"""GPU: every model family of BASELINE.json's configs trains through the
INT8 path (ResNet-20/50 covered elsewhere); checkpoint v2 resumes a run
bit-exactly (params, clip states, LCG stream); the data-parallel phase split
(allreduce hook + int64 wgrad allreduce) is bit-identical to the fused
single-device path at world size 1."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _train(name, batch, steps, seed=3, **kw):
    from paper_1912_12607_b200.layers import int8_replace
    from paper_1912_12607_b200.models import build_model
    from paper_1912_12607_b200.trainer import TrainConfig, Trainer, synthetic_batch
    m = build_model(name, seed=seed)
    int8_replace(m.net)
    tr = Trainer(m, TrainConfig(base_lr=0.02, clip_period=2, seed=11), **kw)
    x, y = synthetic_batch(m, batch, 5)
    reps = [tr.train_step(x, y, it, 100) for it in range(steps)]
    return tr, reps


@pytest.mark.parametrize("name,batch", [("mobilenet_v2", 4), ("inception_v3", 2)])
def test_model_family_trains(name, batch):
    tr, reps = _train(name, batch, 3)
    for r in reps:
        assert not r.diverged and np.isfinite(r.loss)
        assert all(0.1 <= ls.lr_scale <= 1.0 for ls in r.layers)


def test_checkpoint_resume_is_exact(tmp_path):
    from paper_1912_12607_b200.checkpoint import CsvTrace, load_checkpoint, save_checkpoint
    from paper_1912_12607_b200.layers import int8_replace
    from paper_1912_12607_b200.models import build_model
    from paper_1912_12607_b200.trainer import TrainConfig, Trainer, synthetic_batch

    def make():
        m = build_model("resnet20", seed=4)
        int8_replace(m.net)
        return m, Trainer(m, TrainConfig(base_lr=0.05, clip_period=2, seed=9))

    m1, t1 = make()
    x, y = synthetic_batch(m1, 16, 2)
    trace = CsvTrace(str(tmp_path / "trace.csv"))
    for it in range(3):
        trace.report("run", t1.train_step(x, y, it, 50))
    trace.close()
    save_checkpoint(t1, str(tmp_path / "ck.i8ft"), iteration=3)
    r1 = t1.train_step(x, y, 3, 50)
    m2, t2 = make()
    assert load_checkpoint(t2, str(tmp_path / "ck.i8ft")) == 3
    t2.sync_states()
    r2 = t2.train_step(x, y, 3, 50)
    assert r1.loss == r2.loss
    assert torch.equal(t1.pflat, t2.pflat) and int(t1.grad_stream.item()) == int(t2.grad_stream.item())
    lines = open(tmp_path / "trace.csv").read().splitlines()
    assert lines[0] == "run_id,iter,layer,loss,dc,clip,lr_scale,eps_norm,ghat_sqnorm"
    assert len(lines) == 1 + 3 * len(t1.quant_layers)


def test_dp_phase_split_matches_fused_path():
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        ta, ra = _train("resnet20", 16, 3)
        from paper_1912_12607_b200 import ops
        tb, rb = _train("resnet20", 16, 3, force_dp_hook=True)
        for a, b in zip(ra, rb):
            assert a.loss == b.loss
            for la, lb in zip(a.layers, b.layers):
                assert la.clip == lb.clip and la.dc == lb.dc and la.eps_norm == lb.eps_norm
        assert torch.equal(ta.pflat, tb.pflat)
        assert int(ta.grad_stream.item()) == int(tb.grad_stream.item())
        ops.call("i8t_ctx_set_allreduce", ops.ctx(), None, None)
    finally:
        dist.destroy_process_group()
