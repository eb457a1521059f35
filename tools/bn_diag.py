"""Fused vs torch BN: per-leaf forward outputs, backward input-gradients and
parameter gradients after one FP32-mode training step (debug aid for the BN
plumbing).  usage: PYTHONPATH=. python tools/bn_diag.py resnet50 2"""
import sys

import torch

torch.backends.cudnn.allow_tf32 = False
from paper_1912_12607_b200 import layers as L
from paper_1912_12607_b200.models import build_model
from paper_1912_12607_b200.trainer import TrainConfig, Trainer, synthetic_batch

name, batch = sys.argv[1], int(sys.argv[2])
res = {}
impls = (sys.argv[3], sys.argv[4]) if len(sys.argv) > 4 else ("fused", "torch")
for fused in impls:
    L.BN_IMPL = fused
    m = build_model(name, seed=3)
    cfg = TrainConfig(base_lr=0.02, clip_period=2, seed=11)
    cfg.mode = L.Mode.FP32
    tr = Trainer(m, cfg)
    x, y = synthetic_batch(m, batch, 5)
    fw, bw = [], []

    def wrap(layer, path):
        f, b = layer.forward, layer.backward

        def fwd(xx, ctx, f=f, path=path):
            o = f(xx, ctx)
            fw.append((path, L.dense(o).clone()))
            return o

        def bwd(g, ctx, b=b, path=path):
            gin = L.dense_grad(g).clone()
            o = b(g, ctx)
            bw.append((path, gin, None if o is None else L.dense_grad(o).clone()))
            return o
        layer.forward, layer.backward = fwd, bwd

    for path, leaf in L.leaves(m.net):
        wrap(leaf, path)
    r = tr.train_step(x, y, 0, 100)
    grads = {}
    for path, leaf in L.leaves(m.net):
        for p in leaf.params():
            if p.grad is not None:
                grads[f"{path}.{p.name}"] = p.grad.clone()
    res[fused] = (r.loss, fw, bw, grads)


def rel(a, b):
    return float((a - b).abs().max() / (b.abs().max() + 1e-30))


print("loss", res[impls[0]][0], res[impls[1]][0])
print("-- forward (first 3 > 1e-4)")
n = 0
for (p, a), (_, b) in zip(res[impls[0]][1], res[impls[1]][1]):
    if rel(a, b) > 1e-4 and n < 3:
        print(p, "%.3g" % rel(a, b)); n += 1
print("-- backward (first 6 > 1e-4, in backward order)")
n = 0
for (p, gi, go), (_, gi2, go2) in zip(res[impls[0]][2], res[impls[1]][2]):
    di = rel(gi, gi2)
    do = rel(go, go2) if go is not None else 0.0
    if (di > 1e-4 or do > 1e-4) and n < 6:
        print(p, "g_in %.3g g_out %.3g" % (di, do)); n += 1
print("-- param grads > 1e-4:", sum(rel(res[impls[0]][3][k], res[impls[1]][3][k]) > 1e-4 for k in res[impls[0]][3]))
