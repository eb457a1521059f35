"""Step-level CPU restatement of the reference's layer / trainer API --
TEST INFRASTRUCTURE ONLY (the parity checker of the GPU training step; the
product never imports it).

Restates layers.cpp (Conv2d :79-126, Dense :131-225, BatchNorm2d :230-323,
ReLU :328-344, Pool2d :346-415, Sequential :420-435, ResidualBlock :437-469,
InvertedResidual :471-502, SoftmaxCrossEntropy :507-529, int8_replace
:536-546) and train.cpp (Trainer :12-120) in NCHW numpy float32, with the
arithmetic in oracle/oracle.c (sequential double sums in the reference's
order).  EXT geometry (separate stride/pad per dimension, floor-mode output
size, int64 wgrad without the 130000 depth bound) so it also
runs the configs the reference rejects (ResNet-20 b128).

Pinned bit-exactly against the compiled reference Trainer on the nets the
reference accepts (tests/test_oracle_model.py).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import lib as O

F32 = np.float32


def _max(a, b):
    """std::max(a, b) on floats: b if a < b else a."""
    return b if F32(a) < F32(b) else a


@dataclass
class ForwardCtx:
    mode: str = "int8"
    training: bool = True
    track_amax: bool = True
    # teacher(layer, "x", x) -> the input the INT8 layer really sees (teacher
    # forcing with the GPU's values, tests/test_gpu_step_parity.py); None = own value
    teacher: object = None


@dataclass
class BackwardCtx:
    mode: str = "int8"
    iter: int = 0
    stream: list = field(default_factory=lambda: [1])  # [uint32 LCG state], advanced in place
    grid: int = 32
    rounds: int = 2
    clip_search_enabled: bool = True
    clip_period: int = 100
    alpha: float = 20.0
    beta: float = 0.1
    form: str = "exp"
    lr_scaling_enabled: bool = True
    hook: object = None  # optional callback(layer, event, **tensors) -- teacher forcing / capture
    teacher: object = None  # teacher(layer, "g", g) -> the gradient the INT8 layer really sees


class QuantState:
    """QuantState (layers.hpp:28-38)."""

    def __init__(self, period=100):
        self.clip_w = F32(0.0)
        self.clip_a = F32(0.0)
        self.pending_amax = F32(0.0)
        self.cs = O.new_clip_state(period)
        self.dc = 0.0
        self.lr_scale = 1.0
        self.eps_norm = 0.0
        self.ghat_sqnorm = 0.0


def quantize_gradient(qs: QuantState, g: np.ndarray, ctx: BackwardCtx):
    """layers.cpp:19-59.  Returns (q int8, scale)."""
    qs.cs.period = ctx.clip_period
    q, s, stream, st = O.quantize_gradient(qs.cs, g, ctx.iter, ctx.stream[0], ctx.grid, ctx.rounds,
                                           ctx.clip_search_enabled, ctx.lr_scaling_enabled, ctx.alpha, ctx.beta,
                                           ctx.form)
    ctx.stream[0] = stream
    qs.dc, qs.lr_scale, qs.eps_norm, qs.ghat_sqnorm = st["dc"], st["lr_scale"], st["eps_norm"], st["ghat_sqnorm"]
    return q, s


class Layer:
    kind = "layer"
    quantized = False
    qs = None

    def params(self):
        return []

    def buffers(self):
        return []

    def set_quantized(self, on):
        pass

    def visit(self, prefix, fn):
        fn(prefix, self)


class Conv2d(Layer):
    """Conv2d (layers.cpp:79-126), EXT geometry."""

    def __init__(self, in_c, out_c, kernel, stride=1, pad=0, depthwise=False, weight=None):
        kh, kw = (kernel, kernel) if isinstance(kernel, int) else kernel
        self.sh, self.sw = (stride, stride) if isinstance(stride, int) else stride
        self.ph, self.pw = (pad, pad) if isinstance(pad, int) else pad
        self.in_c, self.out_c, self.kh, self.kw, self.depthwise = in_c, out_c, kh, kw, depthwise
        self.kind = "conv_dw" if depthwise else "conv"
        ws = (in_c, 1, kh, kw) if depthwise else (out_c, in_c, kh, kw)
        self.weight = np.zeros(ws, F32) if weight is None else np.array(weight, F32).reshape(ws)
        self.grad_weight = np.zeros(ws, F32)
        self.quantize_enabled = False
        self.qs = QuantState()

    @property
    def quantized(self):
        return self.quantize_enabled

    def set_quantized(self, on):
        self.quantize_enabled = on

    def params(self):
        return [("weight", self.weight, self.grad_weight)]

    def geom(self, x):
        n, c, h, w = x.shape
        if c != self.in_c:
            raise ValueError("Conv2d: bad input shape")
        return O.Geom(n, c, h, w, self.out_c, self.kh, self.kw, self.sh, self.sw, self.ph, self.pw,
                      int(self.depthwise), 1)

    def forward(self, x, ctx: ForwardCtx, hook=None):
        if ctx.teacher:
            x = ctx.teacher(self, "x", x)
        g = self.geom(x)
        self._g = g
        use_int8 = self.quantize_enabled and ctx.mode == "int8"
        qs = self.qs
        if ctx.track_amax:
            qs.pending_amax = _max(qs.pending_amax, O.max_abs(x))
        if not use_int8:
            z = np.empty(O.output_shape(g), F32)
            O._check(O.lib().or_conv_fwd_f32(O.f32(x), O.f32(self.weight), C.byref(g), z))
            return z
        if not qs.clip_w > 0:
            qs.clip_w = _max(O.max_abs(self.weight), F32(1e-12))
        if not qs.clip_a > 0:
            qs.clip_a = _max(O.max_abs(x), F32(1e-12))
        self._qw, _ = O.quantize(self.weight, qs.clip_w)
        self._qa, _ = O.quantize(x, qs.clip_a)
        acc, z = O.conv_fwd(self._qa, self._qw, g, O.quant_scale(qs.clip_a), O.quant_scale(qs.clip_w))
        if hook:
            hook(self, "fwd", x=x, qa=self._qa, qw=self._qw, acc=acc, z=z)
        return z

    def backward(self, g_out, ctx: BackwardCtx):
        if ctx.teacher:
            g_out = ctx.teacher(self, "g", g_out)
        qs = self.qs
        stream_in = ctx.stream[0]
        qg, s_g = quantize_gradient(qs, g_out, ctx)
        g = self._g
        acc_a, ga = O.conv_dgrad(qg, self._qw, g, s_g, O.quant_scale(qs.clip_w))
        acc_w, gw = O.conv_wgrad(qg, self._qa, g, s_g, O.quant_scale(qs.clip_a))
        self.grad_weight[...] = gw
        if ctx.hook:
            ctx.hook(self, "bwd", g=g_out, qg=qg, s_g=s_g, stream_in=stream_in, stream_out=ctx.stream[0],
                     acc_a=acc_a, ga=ga, acc_w=acc_w, gw=gw)
        return ga


class Dense(Layer):
    """Dense (layers.cpp:131-225), INT8 mode; FP32 mode forward for calibration."""
    kind = "fc"

    def __init__(self, in_f, out_f, weight=None):
        self.in_f, self.out_f = in_f, out_f
        self.weight = np.zeros((out_f, in_f), F32) if weight is None else np.array(weight, F32).reshape(out_f, in_f)
        self.bias = np.zeros(out_f, F32)
        self.grad_weight = np.zeros_like(self.weight)
        self.grad_bias = np.zeros_like(self.bias)
        self.quantize_enabled = False
        self.qs = QuantState()

    @property
    def quantized(self):
        return self.quantize_enabled

    def set_quantized(self, on):
        self.quantize_enabled = on

    def params(self):
        return [("weight", self.weight, self.grad_weight), ("bias", self.bias, self.grad_bias)]

    def forward(self, x, ctx: ForwardCtx, hook=None):
        self._in_shape = x.shape
        n = x.shape[0]
        flat = np.ascontiguousarray(x.reshape(n, -1), F32)
        if ctx.teacher:
            flat = ctx.teacher(self, "x", flat)
        if flat.shape[1] != self.in_f:
            raise ValueError("Dense: input does not flatten to expected features")
        use_int8 = self.quantize_enabled and ctx.mode == "int8"
        qs = self.qs
        if ctx.track_amax:
            qs.pending_amax = _max(qs.pending_amax, O.max_abs(flat))
        if not use_int8:
            g = O.Geom(n, self.in_f, 1, 1, self.out_f, 1, 1, 1, 1, 0, 0, 0, 1)
            z = np.empty((n, self.out_f, 1, 1), F32)
            O._check(O.lib().or_conv_fwd_f32(flat, O.f32(self.weight), C.byref(g), z))
            return (z.reshape(n, self.out_f) + self.bias).astype(F32)
        if not qs.clip_w > 0:
            qs.clip_w = _max(O.max_abs(self.weight), F32(1e-12))
        if not qs.clip_a > 0:
            qs.clip_a = _max(O.max_abs(flat), F32(1e-12))
        self._qw, _ = O.quantize(self.weight, qs.clip_w)
        self._qa, _ = O.quantize(flat, qs.clip_a)
        prod = O.gemm_i8(self._qa, np.ascontiguousarray(self._qw.T))
        rescale = float(O.quant_scale(qs.clip_a)) * float(O.quant_scale(qs.clip_w))
        z = (rescale * prod.astype(np.float64)).astype(F32)
        if hook:
            hook(self, "fwd", x=flat, qa=self._qa, qw=self._qw, acc=prod, z=z)
        return (z + self.bias).astype(F32)

    def backward(self, g_out, ctx: BackwardCtx):
        if ctx.teacher:
            g_out = ctx.teacher(self, "g", g_out)
        qs = self.qs
        n = g_out.shape[0]
        stream_in = ctx.stream[0]
        qg, s_g = quantize_gradient(qs, np.ascontiguousarray(g_out, F32), ctx)
        gw = O.gemm_i8(np.ascontiguousarray(qg.T), self._qa)
        self.grad_weight[...] = (float(s_g) * float(O.quant_scale(qs.clip_a)) * gw.astype(np.float64)).astype(F32)
        ga = O.gemm_i8(qg, self._qw)
        g_in = (float(s_g) * float(O.quant_scale(qs.clip_w)) * ga.astype(np.float64)).astype(F32)
        # sum_i s*q[i,o] in double: every partial sum is an exact multiple of s (layers.cpp:216-222)
        self.grad_bias[...] = (qg.astype(np.int64).sum(0).astype(np.float64) * float(s_g)).astype(F32)
        if ctx.hook:
            ctx.hook(self, "bwd", g=g_out, qg=qg, s_g=s_g, stream_in=stream_in, stream_out=ctx.stream[0],
                     acc_a=ga, ga=g_in, acc_w=gw, gw=self.grad_weight.copy())
        return g_in.reshape(self._in_shape)


class BatchNorm2d(Layer):
    """BatchNorm2d (layers.cpp:230-323)."""
    kind = "bn"

    def __init__(self, c, momentum=0.1, eps=1e-5):
        self.c, self.momentum, self.eps = c, momentum, eps
        self.gamma = np.ones(c, F32)
        self.beta = np.zeros(c, F32)
        self.grad_gamma = np.zeros(c, F32)
        self.grad_beta = np.zeros(c, F32)
        self.running_mean = np.zeros(c, F32)
        self.running_var = np.ones(c, F32)

    def params(self):
        return [("gamma", self.gamma, self.grad_gamma), ("beta", self.beta, self.grad_beta)]

    def buffers(self):
        return [("running_mean", self.running_mean), ("running_var", self.running_var)]

    def forward(self, x, ctx, hook=None):
        n, c, h, w = x.shape
        if c != self.c:
            raise ValueError("BatchNorm2d: bad input shape")
        x = O.f32(x)
        y = np.empty_like(x)
        if not ctx.training:
            O.lib().or_bn_forward_eval(x, n, c, h * w, self.gamma, self.beta, self.running_mean, self.running_var,
                                       self.eps, y)
            return y
        self._xhat = np.empty_like(x)
        self._invstd = np.empty(c, np.float64)
        O.lib().or_bn_forward_train(x, n, c, h * w, self.gamma, self.beta, self.running_mean, self.running_var,
                                    self.momentum, self.eps, y, self._xhat, self._invstd)
        if hook:
            hook(self, "fwd", x=x, y=y)
        return y

    def backward(self, g, ctx):
        n, c, h, w = g.shape
        g = O.f32(g)
        gi = np.empty_like(g)
        O.lib().or_bn_backward(g, self._xhat, self._invstd, n, c, h * w, self.gamma, gi, self.grad_gamma,
                               self.grad_beta)
        if ctx.hook:
            ctx.hook(self, "bwd", g=g, gi=gi)
        return gi


class ReLU(Layer):
    """ReLU (layers.cpp:328-344): on = x > 0."""
    kind = "relu"

    def forward(self, x, ctx, hook=None):
        on = x > 0
        if ctx.training:
            self._mask = on
        return np.where(on, x, F32(0.0)).astype(F32)

    def backward(self, g, ctx):
        return np.where(self._mask, g, F32(0.0)).astype(F32)


class Pool2d(Layer):
    """Pool2d (layers.cpp:346-415); EXT padding for max pooling."""

    def __init__(self, kind, k, s, pad=0):
        self.pkind, self.k, self.s, self.pad = (0 if kind == "max" else 1), k, s, pad
        self.kind = "maxpool" if self.pkind == 0 else "avgpool"

    def forward(self, x, ctx, hook=None):
        n, c, h, w = x.shape
        if self.pad == 0 and ((h - self.k) % self.s or (w - self.k) % self.s or h < self.k or w < self.k):
            raise ValueError("Pool2d: geometry does not tile the input")
        oh, ow = (h + 2 * self.pad - self.k) // self.s + 1, (w + 2 * self.pad - self.k) // self.s + 1
        y = np.empty((n, c, oh, ow), F32)
        self._arg = np.zeros((n, c, oh, ow), np.int64)
        O._check(O.lib().or_pool_forward(O.f32(x), n, c, h, w, self.pkind, self.k, self.s, self.pad, y,
                                         self._arg.ctypes.data))
        self._in_shape = x.shape
        return y

    def backward(self, g, ctx):
        n, c, h, w = self._in_shape
        gi = np.empty((n, c, h, w), F32)
        O._check(O.lib().or_pool_backward(O.f32(g), self._arg.ctypes.data, n, c, h, w, self.pkind, self.k, self.s,
                                          self.pad, gi))
        return gi


class Sequential(Layer):
    kind = "sequential"

    def __init__(self, children=None):
        self.children = list(children or [])

    def add(self, name, layer):
        self.children.append((name, layer))
        return layer

    def forward(self, x, ctx, hook=None):
        for _, c in self.children:
            x = c.forward(x, ctx, hook)
        return x

    def backward(self, g, ctx):
        for _, c in reversed(self.children):
            g = c.backward(g, ctx)
        return g

    def visit(self, prefix, fn):
        for name, c in self.children:
            c.visit(f"{prefix}/{name}" if prefix else name, fn)


class ResidualBlock(Layer):
    """ResidualBlock (layers.cpp:437-469): relu(main(x) + shortcut(x)); backward
    main then shortcut, g_main + g_sc."""
    kind = "resblock"

    def __init__(self, main, shortcut=None):
        self.main, self.shortcut, self.relu = main, shortcut, ReLU()

    def forward(self, x, ctx, hook=None):
        m = self.main.forward(x, ctx, hook)
        sc = self.shortcut.forward(x, ctx, hook) if self.shortcut else x
        return self.relu.forward((m + sc).astype(F32), ctx)

    def backward(self, g, ctx):
        g = self.relu.backward(g, ctx)
        gm = self.main.backward(g, ctx)
        gs = self.shortcut.backward(g, ctx) if self.shortcut else g
        return (gm + gs).astype(F32)

    def visit(self, prefix, fn):
        self.main.visit(prefix, fn)
        if self.shortcut:
            self.shortcut.visit(prefix, fn)


class InvertedResidual(Layer):
    """InvertedResidual (layers.cpp:471-502)."""
    kind = "invres"

    def __init__(self, body, use_skip):
        self.body, self.use_skip = body, use_skip

    def forward(self, x, ctx, hook=None):
        y = self.body.forward(x, ctx, hook)
        return (y + x).astype(F32) if self.use_skip else y

    def backward(self, g, ctx):
        gb = self.body.backward(g, ctx)
        return (gb + g).astype(F32) if self.use_skip else gb

    def visit(self, prefix, fn):
        self.body.visit(prefix, fn)


def softmax_ce(logits, labels):
    """SoftmaxCrossEntropy::loss_and_grad (layers.cpp:507-529) -> (loss, g_logits)."""
    logits = O.f32(logits)
    n, k = logits.shape
    g = np.empty_like(logits)
    st = C.c_int()
    loss = O.lib().or_softmax_ce(logits, n, k, np.ascontiguousarray(labels, np.int32), g, C.byref(st))
    O._check(st.value)
    return loss, g


def int8_replace(root) -> int:
    count = [0]

    def fn(_, layer):
        if layer.kind in ("conv", "conv_dw", "fc"):
            layer.set_quantized(True)
            count[0] += 1
    root.visit("", fn)
    return count[0]


def leaves(root):
    out = []
    root.visit("", lambda p, l: out.append((p, l)))
    return out


def named_tensors(root):
    """{"<leaf>.<name>": array} over params and buffers (checkpoint.cpp:50-57)."""
    out = {}
    for path, layer in leaves(root):
        for name, v, _ in layer.params():
            out[f"{path}.{name}"] = v
        for name, v in layer.buffers():
            out[f"{path}.{name}"] = v
    return out


@dataclass
class TrainConfig:
    """TrainConfig (train.hpp:17-32)."""
    mode: str = "int8"
    base_lr: float = 0.1
    schedule: str = "cosine"
    alpha: float = 20.0
    beta: float = 0.1
    form: str = "exp"
    lr_scaling_enabled: bool = True
    grid: int = 32
    rounds: int = 2
    clip_enabled: bool = True
    clip_period: int = 100
    seed: int = 1
    momentum: float = 0.0


class Trainer:
    """Trainer (train.cpp:12-120)."""

    def __init__(self, net, cfg: TrainConfig):
        self.net, self.cfg = net, cfg
        self.stream = [cfg.seed & 0xFFFFFFFF]
        self.leaves = leaves(net)
        self.quant_layers = [(p, l) for p, l in self.leaves if l.qs is not None]
        for _, l in self.quant_layers:
            l.qs.cs.period = cfg.clip_period
        self.mom = {}
        if cfg.momentum != 0.0:
            for i, (_, l) in enumerate(self.leaves):
                for j, (_, v, _) in enumerate(l.params()):
                    self.mom[(i, j)] = np.zeros_like(v)

    def calibrate(self, images):
        self.net.forward(images, ForwardCtx("fp32", False, True))

    def finish_calibration(self):
        self.refresh_wa_clips()

    def refresh_wa_clips(self):
        for _, l in self.quant_layers:
            wmax = F32(0.0)
            for name, v, _ in l.params():
                if name == "weight":
                    wmax = O.max_abs(v)
            if wmax > 0:
                l.qs.clip_w = wmax
            if l.qs.pending_amax > 0:
                l.qs.clip_a = l.qs.pending_amax
            l.qs.pending_amax = F32(0.0)

    def base_lr_at(self, it, total):
        if self.cfg.schedule == "constant" or total <= 0:
            return self.cfg.base_lr
        return self.cfg.base_lr * 0.5 * (1.0 + math.cos(math.pi * (it / total)))

    def train_step(self, images, labels, it, total, fhook=None, bhook=None, teacher=None):
        """Returns {loss, diverged, base_lr_t, layers: [(path, dc, clip, lr_scale, eps, ghat2)], g_logits, logits}.
        teacher: optional teacher-forcing callback (layer, "x" | "g", value) -> value fed to each
        INT8 layer's forward / backward, and (None, "g_logits", g) for the loss gradient."""
        cfg = self.cfg
        rep = dict(iter=it, base_lr_t=self.base_lr_at(it, total), diverged=False)
        logits = self.net.forward(O.f32(images), ForwardCtx(cfg.mode, True, cfg.mode == "int8", teacher), fhook)
        loss, g_logits = softmax_ce(logits, labels)
        if teacher:
            g_logits = teacher(None, "g_logits", g_logits)
        rep.update(loss=loss, logits=logits, g_logits=g_logits)

        def stats():
            rep["layers"] = [(p, l.qs.dc, float(l.qs.cs.clip), l.qs.lr_scale, l.qs.eps_norm, l.qs.ghat_sqnorm)
                             for p, l in self.quant_layers]
            return rep
        if not math.isfinite(loss) or O.has_nonfinite(logits):
            rep["diverged"] = True
            return stats()
        bctx = BackwardCtx(cfg.mode, it, self.stream, cfg.grid, cfg.rounds, cfg.clip_enabled, cfg.clip_period,
                           cfg.alpha, cfg.beta, cfg.form, cfg.lr_scaling_enabled, bhook, teacher)
        self.net.backward(g_logits, bctx)
        for _, l in self.leaves:
            for _, _, gv in l.params():
                if O.has_nonfinite(gv):
                    rep["diverged"] = True
                    return stats()
        for i, (_, l) in enumerate(self.leaves):
            phi = l.qs.lr_scale if (l.qs is not None and cfg.mode == "int8" and l.quantized) else 1.0
            lr = rep["base_lr_t"] * phi
            for j, (_, v, gv) in enumerate(l.params()):
                if cfg.momentum != 0.0:
                    O.lib().or_sgd_momentum_update(v.reshape(-1), O.f32(gv).reshape(-1), self.mom[(i, j)].reshape(-1),
                                                   v.size, lr, cfg.momentum)
                else:
                    O.lib().or_sgd_update(v.reshape(-1), O.f32(gv).reshape(-1), v.size, lr)
        return stats()


# ---------------------------------------------------------------- model builders (reference leaf names)
def build(name, classes=10, side=32):
    """tiny_cnn (models.cpp:22-40), the probe's res_s1 / mbv2_s1
    (oracle/ref_capi.cpp), and resnet20 (EXT geometry; the reference's
    ResidualBlock structure, layers.cpp:437-449)."""
    net = Sequential()
    if name == "tiny_cnn":
        net.add("conv1", Conv2d(3, 4, 3, 1, 1))
        net.add("bn1", BatchNorm2d(4))
        net.add("relu1", ReLU())
        net.add("pool1", Pool2d("max", 2, 2))
        net.add("conv2", Conv2d(4, 8, 3, 1, 1))
        net.add("bn2", BatchNorm2d(8))
        net.add("relu2", ReLU())
        net.add("pool2", Pool2d("max", 2, 2))
        net.add("gap", Pool2d("avg", 8, 8))
        net.add("fc", Dense(8, classes))
        return net
    if name in ("res_s1", "mbv2_s1"):
        net.add("stem", Conv2d(3, 8, 3, 1, 1))
        net.add("stem_bn", BatchNorm2d(8))
        net.add("stem_relu", ReLU())
        if name == "res_s1":
            net.add("block1", res_block(8, 8, 1))
            net.add("block2", res_block(8, 16, 1))
        else:
            net.add("block1", inv_res(8, 12, 1, 2))
            net.add("block2", inv_res(12, 12, 1, 2))
            net.add("head", Conv2d(12, 16, 1, 1, 0))
            net.add("head_bn", BatchNorm2d(16))
            net.add("head_relu", ReLU())
        net.add("gap", Pool2d("avg", side, side))
        net.add("fc", Dense(16, classes))
        return net
    if name == "resnet20":
        net.add("conv1", Conv2d(3, 16, 3, 1, 1))
        net.add("bn1", BatchNorm2d(16))
        net.add("relu1", ReLU())
        cin = 16
        for si, (cout, stride) in enumerate([(16, 1), (32, 2), (64, 2)]):
            for b in range(3):
                s = stride if b == 0 else 1
                net.add(f"stage{si + 1}_block{b + 1}", res_block(cin, cout, s))
                cin = cout
        net.add("gap", Pool2d("avg", 8, 8))
        net.add("fc", Dense(64, classes))
        return net
    raise ValueError(f"unknown model {name}")


def res_block(cin, cout, stride):
    main = Sequential()
    main.add("conv1", Conv2d(cin, cout, 3, stride, 1))
    main.add("bn1", BatchNorm2d(cout))
    main.add("relu1", ReLU())
    main.add("conv2", Conv2d(cout, cout, 3, 1, 1))
    main.add("bn2", BatchNorm2d(cout))
    sc = None
    if stride != 1 or cin != cout:
        sc = Sequential()
        sc.add("conv_sc", Conv2d(cin, cout, 1, stride, 0))
        sc.add("bn_sc", BatchNorm2d(cout))
    return ResidualBlock(main, sc)


def inv_res(cin, cout, stride, expand):
    mid = cin * expand
    body = Sequential()
    body.add("conv1", Conv2d(cin, mid, 1, 1, 0))
    body.add("bn1", BatchNorm2d(mid))
    body.add("relu1", ReLU())
    body.add("conv2", Conv2d(mid, mid, 3, stride, 1, depthwise=True))
    body.add("bn2", BatchNorm2d(mid))
    body.add("relu2", ReLU())
    body.add("conv3", Conv2d(mid, cout, 1, 1, 0))
    body.add("bn3", BatchNorm2d(cout))
    return InvertedResidual(body, stride == 1 and cin == cout)
