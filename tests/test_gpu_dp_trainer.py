"""GPU: the data-parallel Trainer end to end, two ranks sharing cuda:0 over
gloo (NCCL needs one GPU per rank; the box has one).  On a BN-free net (BN is
per-rank by design, so only a BN-free net has a 1-device twin)
two ranks on the batch shards must reproduce one device on the whole batch:
every layer's int8 gradient payload (concatenated over the ranks), the LCG
stream and the parameters after SGD + DCLR bit for bit, the loss to double
rounding -- over DSGC search and non-search steps, with the int64 weight
gradients all-reduced in several buckets.  And bench.py runs under torchrun
with two ranks."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GB, STEPS = 16, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _model():
    from paper_1912_12607_b200.layers import Conv2d, Dense, GlobalAvgPool, ReLU, Sequential, int8_replace
    from paper_1912_12607_b200.models import Model
    gen = torch.Generator().manual_seed(8)
    net = Sequential()
    net.add("conv1", Conv2d(3, 16, 3, 1, 1, gen=gen))
    net.add("relu1", ReLU())
    net.add("conv2", Conv2d(16, 32, 3, 2, 1, gen=gen))
    net.add("relu2", ReLU())
    net.add("conv3", Conv2d(32, 32, 1, 1, 0, gen=gen))
    net.add("relu3", ReLU())
    net.add("pool", GlobalAvgPool())
    net.add("fc", Dense(32, 10, gen=gen))
    int8_replace(net)
    return Model("nobn", net, 10, (3, 16, 16))


def _batch(it):
    g = torch.Generator().manual_seed(100 + it)
    return torch.randn((GB, 16, 16, 3), generator=g), torch.randint(0, 10, (GB,), generator=g)


def _train(rank, world, out):
    from paper_1912_12607_b200 import dp
    from paper_1912_12607_b200 import layers as L
    from paper_1912_12607_b200.trainer import TrainConfig, Trainer
    m = _model()
    tr = Trainer(m, TrainConfig(base_lr=0.05, clip_period=2, seed=21))
    tr.BUCKET_BYTES = 4096  # several int64 buckets
    convs = [getattr(l, "conv", l) for _, l in tr.quant_layers]
    qg = {}
    L.TRACE = lambda conv, ev, **t: qg.__setitem__((ev, convs.index(conv)), t.get("qg")) if ev == "bwd" else None
    res = {"loss": []}
    try:
        for it in range(STEPS):
            x, y = _batch(it)
            if world > 1:
                x, y = dp.shard_batch(x, rank, world), dp.shard_batch(y, rank, world)
            rep = tr.train_step(x.cuda(), y.cuda(), it, 50)
            res["loss"].append(rep.loss)
            for i in range(len(convs)):
                res[f"qg{it}_{i}"] = qg[("bwd", i)].cpu().numpy()
    finally:
        L.TRACE = None
    res["pflat"] = tr.pflat.cpu().numpy()
    res["lcg"] = int(tr.grad_stream.item()) & 0xFFFFFFFF
    np.savez(out, **res)


def _worker(rank, world, port, d):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        _train(rank, world, os.path.join(d, f"r{rank}.npz"))
    finally:
        dist.destroy_process_group()


def test_two_rank_trainer_equals_one_device(tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    _train(0, 1, str(tmp_path / "single.npz"))
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(2)]
    s = np.load(tmp_path / "single.npz")
    for it in range(STEPS):
        i = 0
        while f"qg{it}_{i}" in s:
            np.testing.assert_array_equal(np.concatenate([r[0][f"qg{it}_{i}"], r[1][f"qg{it}_{i}"]]), s[f"qg{it}_{i}"],
                                          err_msg=f"step {it} layer {i}")
            i += 1
        assert i == 4
        for k in range(2):
            assert r[k]["loss"][it] == pytest.approx(s["loss"][it], rel=1e-12)
    for k in range(2):
        np.testing.assert_array_equal(r[k]["pflat"], s["pflat"])
        assert int(r[k]["lcg"]) == int(s["lcg"])


def test_bench_under_torchrun_two_ranks():
    env = dict(os.environ, I8T_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--model",
           "resnet20", "--batch", "32", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["global_batch"] == 64
