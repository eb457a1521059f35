"""GPU: the CUDA-graph replay of the training step (Trainer.train_step_graphed)
is bit-identical to the eager step -- losses, DSGC statistics, parameters and
the LCG stream over search and non-search iterations (search steps and the
first two steps run eagerly; the rest replay), for the identity and the
double-buffered input case."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(graphed, name="resnet20", batch=32, steps=7, period=3):
    from paper_1912_12607_b200.layers import int8_replace
    from paper_1912_12607_b200.models import build_model
    from paper_1912_12607_b200.trainer import TrainConfig, Trainer, synthetic_batch
    m = build_model(name, seed=6)
    int8_replace(m.net)
    tr = Trainer(m, TrainConfig(base_lr=0.05, clip_period=period, seed=13))
    bufs = [synthetic_batch(m, batch, 20 + b) for b in range(2)]
    reps, replays = [], 0
    for it in range(steps):
        x, y = bufs[it % 2]
        if graphed:
            replays += tr.graph_eligible(it)
            reps.append(tr.train_step_graphed(x, y, it, 50, read_stats=True))
        else:
            reps.append(tr.train_step(x, y, it, 50))
    return tr, reps, replays


@pytest.mark.parametrize("name,batch", [("resnet20", 32), ("resnet50", 4)])
def test_graph_replay_equals_eager(name, batch):
    ta, ra, n = _run(True, name, batch)
    tb, rb, _ = _run(False, name, batch)
    assert n >= 3  # some steps really replayed
    for a, b in zip(ra, rb):
        assert a.loss == b.loss and a.diverged == b.diverged
        for la, lb in zip(a.layers, b.layers):
            assert (la.clip, la.dc, la.lr_scale, la.eps_norm) == (lb.clip, lb.dc, lb.lr_scale, lb.eps_norm)
    assert torch.equal(ta.pflat, tb.pflat)
    assert int(ta.grad_stream.item()) == int(tb.grad_stream.item())
