"""Model zoo for the configs of BASELINE.json, built from the reference-style
layers (layers.py): ResNet-20 (CIFAR shape), ResNet-50 (torchvision v1.5
layout: stride on the 3x3), MobileNetV2.  The reference ships only toy nets
(models.cpp:22-89) and cannot express their stride-2 / padded-pool geometry
(SURVEY.md A.3); these use the floor-mode geometry extension.  Weights are
Kaiming-initialised from a seeded generator (synthetic data: no checkpoints).
"""
from __future__ import annotations

import torch

from .layers import (AvgPool2d, BatchNorm2d, Concat, Conv2d, Dense, GlobalAvgPool, InvertedResidual, MaxPool2d, ReLU,
                     ResidualBlock, Sequential)


class Model:
    def __init__(self, name, net, num_classes, in_shape):
        self.name, self.net, self.num_classes, self.in_shape = name, net, num_classes, in_shape


def _cbr(seq, name, cin, cout, k, s, p, gen, dev, relu=True, depthwise=False):
    seq.add(f"{name}", Conv2d(cin, cout, k, s, p, depthwise, gen, dev))
    seq.add(f"{name}_bn", BatchNorm2d(cout, device=dev))
    if relu:
        seq.add(f"{name}_relu", ReLU())


def _chain_blocks(net):
    """Tell each ResidualBlock which conv consumes its output next (its int8
    input is then written by the block's BN + residual + ReLU pass)."""
    blocks = [layer for _, layer in net.children if isinstance(layer, ResidualBlock)]
    for a, b in zip(blocks, blocks[1:]):
        first = b.main.children[0][1] if b.main.children else None
        if isinstance(first, Conv2d):
            a.next_conv = first


def resnet20(num_classes=10, seed=1, device="cuda") -> Model:
    gen = torch.Generator().manual_seed(seed)
    net = Sequential()
    _cbr(net, "conv1", 3, 16, 3, 1, 1, gen, device)
    cin = 16
    for si, (cout, stride) in enumerate([(16, 1), (32, 2), (64, 2)]):
        for b in range(3):
            s = stride if b == 0 else 1
            main = Sequential()
            _cbr(main, "conv1", cin, cout, 3, s, 1, gen, device)
            _cbr(main, "conv2", cout, cout, 3, 1, 1, gen, device, relu=False)
            sc = None
            if s != 1 or cin != cout:
                sc = Sequential()
                _cbr(sc, "conv_sc", cin, cout, 1, s, 0, gen, device, relu=False)
            net.add(f"stage{si + 1}_block{b + 1}", ResidualBlock(main, sc))
            cin = cout
    net.add("pool", GlobalAvgPool())
    net.add("fc", Dense(64, num_classes, gen, device))
    _chain_blocks(net)
    return Model("resnet20", net, num_classes, (3, 32, 32))


def resnet50(num_classes=1000, seed=1, device="cuda") -> Model:
    gen = torch.Generator().manual_seed(seed)
    net = Sequential()
    _cbr(net, "conv1", 3, 64, 7, 2, 3, gen, device)
    net.add("maxpool", MaxPool2d(3, 2, 1))
    cin = 64
    for li, (width, blocks, stride) in enumerate([(64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)]):
        for b in range(blocks):
            s = stride if b == 0 else 1
            main = Sequential()
            _cbr(main, "conv1", cin, width, 1, 1, 0, gen, device)
            _cbr(main, "conv2", width, width, 3, s, 1, gen, device)
            _cbr(main, "conv3", width, width * 4, 1, 1, 0, gen, device, relu=False)
            sc = None
            if b == 0:
                sc = Sequential()
                _cbr(sc, "downsample", cin, width * 4, 1, s, 0, gen, device, relu=False)
            net.add(f"layer{li + 1}_{b}", ResidualBlock(main, sc))
            cin = width * 4
    net.add("pool", GlobalAvgPool())
    net.add("fc", Dense(2048, num_classes, gen, device))
    _chain_blocks(net)
    return Model("resnet50", net, num_classes, (3, 224, 224))


def mobilenet_v2(num_classes=1000, seed=1, device="cuda", width_mult=1.0) -> Model:
    gen = torch.Generator().manual_seed(seed)
    net = Sequential()
    _cbr(net, "conv1", 3, 32, 3, 2, 1, gen, device)
    cin = 32
    cfg = [(1, 16, 1, 1), (6, 24, 2, 2), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]
    bi = 0
    for t, c, n, s in cfg:
        for i in range(n):
            stride = s if i == 0 else 1
            mid = cin * t
            body = Sequential()
            if t != 1:
                _cbr(body, "expand", cin, mid, 1, 1, 0, gen, device)
            _cbr(body, "dw", mid, mid, 3, stride, 1, gen, device, depthwise=True)
            _cbr(body, "project", mid, c, 1, 1, 0, gen, device, relu=False)
            net.add(f"block{bi}", InvertedResidual(body, stride == 1 and cin == c))
            cin = c
            bi += 1
    _cbr(net, "conv_last", cin, 1280, 1, 1, 0, gen, device)
    net.add("pool", GlobalAvgPool())
    net.add("fc", Dense(1280, num_classes, gen, device))
    return Model("mobilenet_v2", net, num_classes, (3, 224, 224))


def _basic(cin, cout, k, s=1, p=0, gen=None, dev="cuda"):
    seq = Sequential()
    _cbr(seq, "conv", cin, cout, k, s, p, gen, dev)
    return seq


def _chain(specs, gen, dev):
    """specs: list of (cin, cout, kernel, stride, pad) conv-bn-relu units."""
    seq = Sequential()
    for i, (ci, co, k, s, p) in enumerate(specs):
        _cbr(seq, f"conv{i}", ci, co, k, s, p, gen, dev)
    return seq


def _pool_branch(pool, cin, cout, gen, dev):
    seq = Sequential()
    seq.add("pool", pool)
    if cout:
        _cbr(seq, "conv", cin, cout, 1, 1, 0, gen, dev)
    return seq


def inception_v3(num_classes=1000, seed=1, device="cuda") -> Model:
    """InceptionV3 (torchvision layout, no aux head) at 299x299: 94 convs incl.
    the asymmetric 1x7 / 7x1 / 1x3 / 3x1 kernels with (0,3)/(3,0)/(0,1)/(1,0)
    padding that the reference's single-pad geometry cannot express (A.3-2)."""
    g, d = torch.Generator().manual_seed(seed), device
    net = Sequential()
    for name, (ci, co, k, s, p) in [("c1a", (3, 32, 3, 2, 0)), ("c2a", (32, 32, 3, 1, 0)), ("c2b", (32, 64, 3, 1, 1))]:
        _cbr(net, name, ci, co, k, s, p, g, d)
    net.add("pool1", MaxPool2d(3, 2))
    _cbr(net, "c3b", 64, 80, 1, 1, 0, g, d)
    _cbr(net, "c4a", 80, 192, 3, 1, 0, g, d)
    net.add("pool2", MaxPool2d(3, 2))
    cin = 192
    for i, pf in enumerate((32, 64, 64)):  # InceptionA x3
        net.add(f"mixed5{'bcd'[i]}", Concat([
            _basic(cin, 64, 1, gen=g, dev=d),
            _chain([(cin, 48, 1, 1, 0), (48, 64, 5, 1, 2)], g, d),
            _chain([(cin, 64, 1, 1, 0), (64, 96, 3, 1, 1), (96, 96, 3, 1, 1)], g, d),
            _pool_branch(AvgPool2d(3, 1, 1), cin, pf, g, d)]))
        cin = 224 + pf
    net.add("mixed6a", Concat([  # InceptionB
        _basic(cin, 384, 3, 2, 0, g, d),
        _chain([(cin, 64, 1, 1, 0), (64, 96, 3, 1, 1), (96, 96, 3, 2, 0)], g, d),
        _pool_branch(MaxPool2d(3, 2), cin, 0, g, d)]))
    cin = 768
    for i, c7 in enumerate((128, 160, 160, 192)):  # InceptionC x4
        net.add(f"mixed6{'bcde'[i]}", Concat([
            _basic(cin, 192, 1, gen=g, dev=d),
            _chain([(cin, c7, 1, 1, 0), (c7, c7, (1, 7), 1, (0, 3)), (c7, 192, (7, 1), 1, (3, 0))], g, d),
            _chain([(cin, c7, 1, 1, 0), (c7, c7, (7, 1), 1, (3, 0)), (c7, c7, (1, 7), 1, (0, 3)),
                    (c7, c7, (7, 1), 1, (3, 0)), (c7, 192, (1, 7), 1, (0, 3))], g, d),
            _pool_branch(AvgPool2d(3, 1, 1), cin, 192, g, d)]))
    net.add("mixed7a", Concat([  # InceptionD
        _chain([(768, 192, 1, 1, 0), (192, 320, 3, 2, 0)], g, d),
        _chain([(768, 192, 1, 1, 0), (192, 192, (1, 7), 1, (0, 3)), (192, 192, (7, 1), 1, (3, 0)),
                (192, 192, 3, 2, 0)], g, d),
        _pool_branch(MaxPool2d(3, 2), 768, 0, g, d)]))
    cin = 1280
    for i in range(2):  # InceptionE x2
        b3 = Sequential()
        _cbr(b3, "conv", cin, 384, 1, 1, 0, g, d)
        b3.add("split", Concat([_basic(384, 384, (1, 3), 1, (0, 1), g, d), _basic(384, 384, (3, 1), 1, (1, 0), g, d)]))
        bd = _chain([(cin, 448, 1, 1, 0), (448, 384, 3, 1, 1)], g, d)
        bd.add("split", Concat([_basic(384, 384, (1, 3), 1, (0, 1), g, d), _basic(384, 384, (3, 1), 1, (1, 0), g, d)]))
        net.add(f"mixed7{'bc'[i]}", Concat([_basic(cin, 320, 1, gen=g, dev=d), b3, bd,
                                            _pool_branch(AvgPool2d(3, 1, 1), cin, 192, g, d)]))
        cin = 2048
    net.add("pool", GlobalAvgPool())
    net.add("fc", Dense(2048, num_classes, g, d))
    return Model("inception_v3", net, num_classes, (3, 299, 299))


MODELS = {"resnet20": resnet20, "resnet50": resnet50, "mobilenet_v2": mobilenet_v2, "inception_v3": inception_v3}


def build_model(name: str, seed: int = 1, device="cuda", **kw) -> Model:
    """build_model (models.hpp:24-25)."""
    if name not in MODELS:
        raise ValueError(f"unknown model {name}")
    return MODELS[name](seed=seed, device=device, **kw)


def conv_gop_per_image(model: Model) -> float:
    """2*N*K*P*Q*(C/groups)*R*S ops per pass summed over quantised conv/fc
    layers x 3 passes (fwd, dgrad, wgrad), per image, minus the
    first conv's dgrad (the image gradient is never computed): 24.299 GOP for
    ResNet-50 at 224x224."""
    c, h, w = model.in_shape
    total = 0.0

    def walk(layer, shape):
        nonlocal total
        from . import layers as L
        if isinstance(layer, L.Sequential):
            for _, ch in layer.children:
                shape = walk(ch, shape)
            return shape
        if isinstance(layer, L.ResidualBlock):
            out = walk(layer.main, shape)
            if layer.shortcut:
                walk(layer.shortcut, shape)
            return out
        if isinstance(layer, L.InvertedResidual):
            return walk(layer.body, shape)
        if isinstance(layer, L.Concat):
            outs = [walk(b, shape) for b in layer.branches]
            return outs[0][:3] + (sum(o[3] for o in outs),)
        if isinstance(layer, L.AvgPool2d):
            n, hh, ww, cc = shape
            return (n, (hh + 2 * layer.p - layer.k) // layer.s + 1, (ww + 2 * layer.p - layer.k) // layer.s + 1, cc)
        if isinstance(layer, L.Conv2d):
            n, hh, ww, cc = shape
            p = (hh + 2 * layer.ph - layer.kh) // layer.sh + 1
            q = (ww + 2 * layer.pw - layer.kw) // layer.sw + 1
            cin = 1 if layer.depthwise else cc
            if not layer.depthwise and cc != layer.in_c:
                raise ValueError(f"channel mismatch in model walk: {cc} vs {layer.in_c}")
            # fwd + wgrad always; dgrad unless the layer's input gradient is discarded (the stem)
            passes = 3 if layer.need_input_grad and not first[0] else 2
            first[0] = False
            total += passes * 2.0 * p * q * layer.out_c * cin * layer.kh * layer.kw
            return (n, p, q, layer.out_c)
        if isinstance(layer, L.Dense):
            total += 3 * 2.0 * layer.in_f * layer.out_f
            return (shape[0], layer.out_f)
        if isinstance(layer, L.MaxPool2d):
            n, hh, ww, cc = shape
            return (n, (hh + 2 * layer.p - layer.k) // layer.s + 1, (ww + 2 * layer.p - layer.k) // layer.s + 1, cc)
        if isinstance(layer, L.GlobalAvgPool):
            return (shape[0], shape[3])
        return shape

    first = [True]
    walk(model.net, (1, h, w, c))
    return total / 1e9
