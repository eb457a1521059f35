"""Layer API of the INT8 training path on the device -- the reference's
Layer / Conv2d / Dense / BatchNorm2d / ReLU / Pool2d / Sequential /
ResidualBlock / InvertedResidual / SoftmaxCrossEntropy (layers.hpp:69-255,
layers.cpp:19-546) with explicit forward/backward, so that the backward order
-- and with it the order in which the single LCG gradient stream is consumed
(train.cpp:13, layers.cpp:426-430, 458-464) -- is the reference's.

Activations travel as NHWC-contiguous float32 CUDA tensors [N, H, W, C].  The
quantised conv / fc layers (Conv2d, Dense) run entirely through the C-ABI of
libi8t_cuda.so: nearest quantisation of W and a with fused amax tracking,
the tcgen05 implicit-GEMM forward, the fused DSGC + stochastic gradient
quantiser, tcgen05 backward-data / backward-weight.  FP32 layers (BN, ReLU,
pooling, softmax-CE) are outside the graded path and use
PyTorch/cuDNN library ops.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from enum import Enum

import torch
import torch.nn.functional as F

from . import ops
from ._lib import ConvGeom, DsgcView, call


class Mode(Enum):
    FP32 = 0
    INT8 = 1


@dataclass
class ForwardCtx:
    """ForwardCtx (layers.hpp:40-45)."""
    mode: Mode = Mode.INT8
    training: bool = True
    track_amax: bool = True
    weights_quantized: bool = False  # the trainer already ran i8t_quantize_weights_multi for this step


@dataclass
class BackwardCtx:
    """BackwardCtx (layers.hpp:55-67); grad_stream is the device LCG state."""
    mode: Mode = Mode.INT8
    iter: int = 0
    grad_stream: torch.Tensor | None = None
    grid_resolution: int = 32
    refine_rounds: int = 2
    clip_search_enabled: bool = True
    clip_period: int = 100
    alpha: float = 20.0
    beta: float = 0.1
    form: str = "exp"
    lr_scaling_enabled: bool = True
    wgrad_allreduce: object = None  # callable(int64 acc tensor) -> async work, data parallelism (exact sum)
    # (work, finalize) pairs: the int64 weight-gradient allreduces run while the
    # backward continues; the trainer waits on each and rescales before the update
    deferred: list = field(default_factory=list)
    # single device: weight gradients on this side stream (their own i8t_ctx),
    # overlapping the backward-data chain; the trainer joins it before the update
    wgrad_stream: object = None


@dataclass
class ParamRef:
    name: str
    value: torch.Tensor
    grad: torch.Tensor | None


# ------------------------------------------------------------------ lazy values
# BN + ReLU are fused into the INT8 path's HBM passes (csrc/bnfuse.cu): a BN
# forward returns LazyAct (act(bn(z)) not materialised), which the next
# Conv2d quantises in one pass; a BN backward returns BnGrad, which the
# previous Conv2d feeds straight into the stochastic gradient quantiser.  Any
# other consumer calls dense() / dense_grad() and gets a plain tensor.
# "fused" (default): lazy values as above; "eager": the same kernels with every
# value materialised at once (bit-identical results, used to test the
# plumbing); "torch": torch's fp32 batch norm.
BN_IMPL = os.environ.get("I8T_BN", "fused")
# residual joins inside the dgrad epilogue (I8T_JOIN=1; identity joins take the
# block ReLU mask as packed bits).  Off by default: the addend loads sit on the
# epilogue's critical path (its 96-register budget leaves no room to prefetch
# them) and measured slower: 37.7 vs 35.7 ms per ResNet-50 b256 step (B200).
JOIN_FUSION = os.environ.get("I8T_JOIN", "0") == "1"
# The projection-shortcut join (the downsample conv's dgrad adds the
# main-branch gradient; 4 ResNet-50 blocks) pays off: 35.01 -> 34.90 ms per
# step.  I8T_JOIN_PROJ=0 turns it off.
JOIN_PROJ = os.environ.get("I8T_JOIN_PROJ", "1") == "1" or JOIN_FUSION
# The identity-shortcut join (gm + g * mask) materialised inside the preceding
# BatchNorm's backward column-sum pass instead of its own elementwise pass
# (JoinGrad; g_out is written once and never re-read by the reduction).
# I8T_JOIN_REDUCE=0 keeps the separate i8t_add_masked_bits.
JOIN_REDUCE = os.environ.get("I8T_JOIN_REDUCE", "1") == "1"
# The projection block's shortcut BN reduces its backward sums in the main
# branch's last-BN pass over the same joined gradient (i8t_bn_bwd_reduce_join2).
JOIN_REDUCE2 = os.environ.get("I8T_JOIN_REDUCE2", "1") == "1"
# The projection shortcut conv reuses the block's first conv's int8 input when
# their activation clips agree (i8t_quantize_nearest_shared).  I8T_SHARE_ACT=0
# quantises twice.
SHARE_ACT = os.environ.get("I8T_SHARE_ACT", "1") == "1"
# Test instrumentation: when set, TRACE(conv, event, **tensors) is called at the
# end of every INT8 Conv2d forward ("fwd") and backward ("bwd") -- the step-level
# parity test (tests/test_gpu_step_parity.py) teacher-forces the CPU oracle with
# these values.  None in production (one attribute test per call).
TRACE = None


class LazyAct:
    """act(bn(z)) with z the NHWC conv output and `bn` its BatchNorm2d layer."""

    def __init__(self, z, bn, relu=False):
        self.z, self.bn, self.relu = z, bn, relu

    @property
    def shape(self):
        return self.z.shape

    @property
    def device(self):
        return self.z.device

    def numel(self):
        return self.z.numel()

    def materialize(self, res=None, quant_for=None, ctx=None, mask_bits=None):
        """y = act(bn(z) [+ res]).  With quant_for = the conv that consumes y next
        (and its clip known), the same pass also writes that conv's int8 input
        (attached as y._i8t_q, picked up by Conv2d.forward)."""
        n, h, w, c = self.z.shape
        y = torch.empty_like(self.z)
        r, rz, rbn = (None, None, None)
        if isinstance(res, LazyAct):
            rz, rbn = res.z, res.bn
        elif res is not None:
            r = res
        args = (ops.ctx(), ops._p(self.z), n * h * w, c, ops._p(self.bn.stats), ops._p(self.bn.gamma),
                ops._p(self.bn.beta), int(self.relu), ops._p(r), ops._p(rz), ops._p(rbn.stats) if rbn else None,
                ops._p(rbn.gamma) if rbn else None, ops._p(rbn.beta) if rbn else None, ops._p(y))
        conv = quant_for
        pre = conv is not None and ctx is not None and conv.takes_prequantized(c, ctx)
        if pre or mask_bits is not None:
            q = torch.empty((n, h, w, c), dtype=torch.int8, device=y.device) if pre else None
            qs = conv.qs if pre else None
            call("i8t_bn_act_q", *args, ops._p(qs.clip_a) if pre else None, ops._p(q),
                 ops._p(qs.pending_amax) if pre and ctx.track_amax else None, ops._p(mask_bits))
            if pre:
                y._i8t_q = (conv, q)
        else:
            call("i8t_bn_act", *args)
        return y


class MaskedGrad:
    """g * mask: mode 1 = ReLU mask of act(bn(z)) of `bn`, mode 2 = (mask_y > 0)."""

    def __init__(self, g, mode, bn=None, mask_y=None):
        self.g, self.mode, self.bn, self.mask_y = g, mode, bn, mask_y

    @property
    def shape(self):
        return self.g.shape

    @property
    def device(self):
        return self.g.device

    def numel(self):
        return self.g.numel()

    def materialize(self):
        g = dense_grad(self.g)
        if self.mode == 2:
            return torch.where(self.mask_y > 0, g, torch.zeros((), device=g.device))
        if self.mode == 3:
            return torch.where(unpack_mask(self.mask_y, g.numel()).view_as(g), g, torch.zeros((), device=g.device))
        y = LazyAct(self.bn._z, self.bn, relu=True).materialize()
        return torch.where(y > 0, g, torch.zeros((), device=g.device))


class BnGrad:
    """BN backward of (g, mask) not yet materialised (sums already reduced)."""

    def __init__(self, g, bn, mode, mask_y):
        self.g, self.bn, self.mode, self.mask_y = g, bn, mode, mask_y

    @property
    def shape(self):
        return self.g.shape

    @property
    def device(self):
        return self.g.device

    def numel(self):
        return self.g.numel()

    def materialize(self, stats=None):
        n, h, w, c = self.g.shape
        out = torch.empty_like(self.g)
        if stats is not None:  # + max|g|, non-finite count, sum g^2 of the result (a DSGC search's first pass)
            call("i8t_bn_bwd_apply_stats", ops.ctx(), ops._p(self.g), ops._p(self.bn._z), n * h * w, c,
                 ops._p(self.bn.stats), ops._p(self.bn.gamma), ops._p(self.bn.beta), self.mode, ops._p(self.mask_y),
                 ops._p(out), ops._p(stats))
            return out
        call("i8t_bn_bwd_apply", ops.ctx(), ops._p(self.g), ops._p(self.bn._z), n * h * w, c, ops._p(self.bn.stats),
             ops._p(self.bn.gamma), ops._p(self.bn.beta), self.mode, ops._p(self.mask_y), ops._p(out))
        return out


class JoinGrad:
    """gm + g * bit: the identity-shortcut join of a residual block's backward
    (layers.cpp:458-464) not yet materialised.  The preceding BatchNorm's
    backward materialises it inside its column-sum pass
    (i8t_bn_bwd_reduce_join); anything else calls materialize()."""

    def __init__(self, gm, g, bits):
        self.gm, self.g, self.bits = gm, g, bits
        self.out = None
        self.co_bn = None  # a second BN reduced on the same masked gradient in the same pass (projection shortcut)

    @property
    def shape(self):
        return self.g.shape

    @property
    def device(self):
        return self.g.device

    def numel(self):
        return self.g.numel()

    def materialize(self):
        if self.out is None:
            out = torch.empty_like(self.gm)
            call("i8t_add_masked_bits", ops.ctx(), ops._p(self.gm), ops._p(self.g), ops._p(self.bits), self.gm.numel(),
                 ops._p(out))
            self.out = out
            self.gm = self.g = self.bits = None
        return self.out


def unpack_mask(bits: torch.Tensor, n: int) -> torch.Tensor:
    """Packed ReLU mask (int32 words, bit e%32 of word e/32) -> bool [n]."""
    sh = torch.arange(32, device=bits.device, dtype=torch.int32)
    return ((bits.view(-1, 1) >> sh) & 1).view(-1)[:n].bool()


def dense(x):
    return x.materialize() if isinstance(x, LazyAct) else x


def dense_grad(g):
    return g.materialize() if isinstance(g, (MaskedGrad, BnGrad, JoinGrad)) else g


# ------------------------------------------------------------------ state arena
class StateArena:
    """All per-layer device state in one buffer so a step reads every layer's
    DSGC view with a single D2H copy.  Per layer: one DsgcState (clip.hpp:12-18
    + QuantState measurements) and a float block [clip_w, clip_a,
    pending_amax, tmp] (QuantState, layers.hpp:28-38)."""

    def __init__(self, device="cuda"):
        self.dsgc_size = (int(ops.lib().i8t_dsgc_state_size()) + 63) // 64 * 64
        self.layers = []
        self.device = device
        self.buf = None

    def register(self, layer) -> int:
        self.layers.append(layer)
        return len(self.layers) - 1

    def build(self, period: int):
        n = len(self.layers)
        self.slot = self.dsgc_size + 64
        self.buf = torch.zeros(n * self.slot, dtype=torch.uint8, device=self.device)
        for i, layer in enumerate(self.layers):
            base = i * self.slot
            layer.qs.bind(self, self.buf[base: base + self.dsgc_size],
                          self.buf[base + self.dsgc_size: base + self.slot].view(torch.float32), period)

    def read_views(self) -> list[DsgcView]:
        host = self.buf.cpu()  # one D2H copy (syncs the stream)
        out = []
        for i in range(len(self.layers)):
            b = bytes(host[i * self.slot: i * self.slot + C.sizeof(DsgcView)].numpy())
            out.append(DsgcView.from_buffer_copy(b))
        return out


class QuantState:
    """QuantState (layers.hpp:28-38) on the device: DsgcState + [clip_w,
    clip_a, pending_amax, tmp], with host mirrors that decide lazily
    initialised clips and Periodic-Update due-ness without syncing."""

    def __init__(self):
        self.dsgc = None
        self.f = None
        self.clip_w_set = False
        self.clip_a_set = False
        self.layer_id = ""

    def bind(self, arena, dsgc_bytes, floats, period):
        self.dsgc = _ArenaDsgc(dsgc_bytes, period, self.layer_id)
        self.f = floats
        self.f.zero_()

    @property
    def clip_w(self):
        return self.f[0:1]

    @property
    def clip_a(self):
        return self.f[1:2]

    @property
    def pending_amax(self):
        return self.f[2:3]

    @property
    def tmp(self):
        return self.f[3:4]


class _ArenaDsgc(ops.DsgcState):
    """ops.DsgcState living inside the StateArena buffer."""

    def __init__(self, buf, period, layer_id):  # noqa: super().__init__ allocates; we adopt the slice instead
        self.buf = buf
        self.layer_id = layer_id
        self.period = period
        call("i8t_dsgc_init", ops.ctx(), ops._p(self.buf), period)
        self.iter_of_last_update = -1
        self.clip_valid = False

    def clip_q_ptr(self):
        """Device float holding the clip of the last quantised gradient."""
        return self.buf[_CLIP_Q_OFF:_CLIP_Q_OFF + 4].view(torch.float32)


_CLIP_Q_OFF = DsgcView.clip_q.offset
_SCALE_OFF = DsgcView.scale.offset


# ------------------------------------------------------------------ layers
class Layer:
    kind = "layer"

    def forward(self, x, ctx: ForwardCtx):
        raise NotImplementedError

    def backward(self, g, ctx: BackwardCtx):
        raise NotImplementedError

    def params(self) -> list[ParamRef]:
        return []

    def param_attrs(self) -> list[tuple]:
        """(owner, value attribute, grad attribute) per parameter, in params() order."""
        return []

    def buffers(self) -> list[ParamRef]:
        return []

    quantized = False
    qs: QuantState | None = None

    def set_quantized(self, on: bool):
        pass

    def visit(self, prefix, fn):
        fn(prefix, self)


def _dp_max_(t: torch.Tensor):
    """MAX all-reduce across data-parallel ranks (no-op on one process)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)


def _fp32_exact():
    """FP32-mode convolutions (calibration, the FP32 baseline; conv2d_f32 in the
    reference) in IEEE fp32, not TF32: cuDNN's default TF32 inputs would shift
    the activation maxima the calibration hands to the INT8 clips."""
    return torch.backends.cudnn.flags(enabled=True, benchmark=False, deterministic=False, allow_tf32=False)


def _kaiming(shape, fan_in, gen, device):
    return (torch.randn(shape, generator=gen, device="cpu") * math.sqrt(2.0 / fan_in)).to(device)


class Conv2d(Layer):
    """INT8 convolution layer (layers.hpp:86-115, layers.cpp:65-126) with
    separate (kh, kw), stride and padding per dimension (EXT)."""

    def __init__(self, in_c, out_c, kernel, stride=1, pad=0, depthwise=False, gen=None, device="cuda"):
        kh, kw = (kernel, kernel) if isinstance(kernel, int) else kernel
        sh, sw = (stride, stride) if isinstance(stride, int) else stride
        ph, pw = (pad, pad) if isinstance(pad, int) else pad
        if depthwise and in_c != out_c:
            raise ValueError("Conv2d: depthwise needs in_c == out_c")
        self.in_c, self.out_c, self.kh, self.kw = in_c, out_c, kh, kw
        self.sh, self.sw, self.ph, self.pw, self.depthwise = sh, sw, ph, pw, depthwise
        self.kind = "conv_dw" if depthwise else "conv"
        fan_in = (1 if depthwise else in_c) * kh * kw
        ws = (in_c, 1, kh, kw) if depthwise else (out_c, in_c, kh, kw)
        self.weight = _kaiming(ws, fan_in, gen or torch.Generator().manual_seed(0), device)
        self.grad_weight = torch.zeros_like(self.weight)
        self.quantize_enabled = False
        self.qs = QuantState()
        self.c_pad = in_c if depthwise else ops.pad4(in_c)
        self.k_pad = ops.pad4(out_c)
        self.ld_w = ops.pad16(kh * kw * self.c_pad)
        self.ld_wt = ops.pad16(kh * kw * self.k_pad)
        self._qw = self._qwt = None
        self.wgrad_acc = None
        self.keep_qg = False  # Dense needs the int8 gradient for its bias
        self._qg = None
        self.need_input_grad = True  # False for the first layer: the image gradient is discarded
        # residual join handed down by a ResidualBlock: (add_g, add_y) -> the
        # dgrad epilogue returns dgrad + add_g [* (add_y > 0)]; join_done reports it
        self.dgrad_join = None
        self.join_done = False
        self.act_twin = None  # a conv quantising the same input first (ResidualBlock: the shortcut's twin)
        self.keep_qa_src = False  # this conv is someone's act_twin: remember which tensor _qa quantised
        self._qa_src = None

    @property
    def quantized(self):
        return self.quantize_enabled

    def set_quantized(self, on):
        self.quantize_enabled = on

    def wq_desc(self):
        """(w, clip, q_krsc, q_crsk, k, c, rs, c_pad, ld_krsc, k_pad, ld_crsk, src_krsc) of
        i8t_wq_desc once the buffers and clip exist, else None."""
        if self._qw is None or not self.qs.clip_w_set:
            return None
        rs = self.kh * self.kw
        if self.depthwise:
            return (self.weight, self.qs.clip_w, self._qw, None, self.in_c, 1, rs, 1, rs, 0, 0, 0)
        return (self.weight, self.qs.clip_w, self._qw, self._qwt, self.out_c, self.in_c, rs, self.c_pad, self.ld_w,
                self.k_pad, self.ld_wt, 0)

    def takes_prequantized(self, c, ctx) -> bool:
        """Can the producer of this conv's input quantise it (clip known, no channel padding)?"""
        return (self.quantize_enabled and ctx.mode == Mode.INT8 and self.qs.clip_a_set and not self.depthwise
                and self.c_pad == c == self.in_c)

    def params(self):
        return [ParamRef("weight", self.weight, self.grad_weight)]

    def param_attrs(self):
        return [(self, "weight", "grad_weight")]

    def geom(self, x):
        n, h, w, c = x.shape
        if c != self.in_c:
            raise ValueError(f"Conv2d: bad input shape {tuple(x.shape)}")
        return ConvGeom(n, c, h, w, self.out_c, self.kh, self.kw, self.sh, self.sw, self.ph, self.pw,
                        int(self.depthwise), 1)

    # -- forward (layers.cpp:98-111)
    def forward(self, x, ctx: ForwardCtx):
        g = self.geom(x)
        self._geom = g
        p, q = g.out_hw()
        use_int8 = self.quantize_enabled and ctx.mode == Mode.INT8
        h = ops.ctx()
        qs = self.qs
        fuse_in = (isinstance(x, LazyAct) and use_int8 and qs.clip_a_set and not self.depthwise
                   and self.c_pad == self.in_c)
        if not fuse_in:
            x = dense(x)
        if not use_int8:
            if ctx.track_amax:
                call("i8t_max_abs", h, ops._p(x), x.numel(), ops._p(qs.tmp))
                torch.maximum(qs.pending_amax, qs.tmp, out=qs.pending_amax)
            if ctx.training:
                self._x = x
            xc = x.permute(0, 3, 1, 2)
            with _fp32_exact():
                y = F.conv2d(xc, self.weight, None, (self.sh, self.sw), (self.ph, self.pw),
                             groups=self.in_c if self.depthwise else 1)
            return y.permute(0, 2, 3, 1).contiguous()
        # lazy clip init: clip = max(max_abs(t), 1e-12) (layers.cpp:106-107); under data
        # parallelism the max is over the global batch, so every rank quantises with one scale
        if not qs.clip_w_set:
            call("i8t_max_abs", h, ops._p(self.weight), self.weight.numel(), ops._p(qs.clip_w))
            qs.clip_w.clamp_(min=1e-12)
            _dp_max_(qs.clip_w)
            qs.clip_w_set = True
        if not qs.clip_a_set and not fuse_in:
            call("i8t_max_abs", h, ops._p(x), x.numel(), ops._p(qs.clip_a))
            qs.clip_a.clamp_(min=1e-12)
            _dp_max_(qs.clip_a)
            qs.clip_a_set = True
        # weights -> KRSC (fwd) + CRSK (dgrad) int8 in one pass (or all layers at once, see wq_desc)
        if self.depthwise:
            if self._qw is None:
                self._qw = torch.zeros((self.in_c, self.kh * self.kw), dtype=torch.int8, device=x.device)
            if not ctx.weights_quantized:
                call("i8t_quantize_nearest", h, ops._p(self.weight), self.weight.numel(), ops._p(qs.clip_w),
                     ops._p(self._qw), None, 0)
        else:
            if self._qw is None:  # zeroed once: the padding bytes are never written
                self._qw = torch.zeros((self.out_c, self.ld_w), dtype=torch.int8, device=x.device)
                self._qwt = torch.zeros((self.in_c, self.ld_wt), dtype=torch.int8, device=x.device)
            if not ctx.weights_quantized:
                call("i8t_quantize_weight", h, ops._p(self.weight), 0, self.out_c, self.in_c, self.kh, self.kw,
                     ops._p(qs.clip_w), ops._p(self._qw), self.c_pad, self.ld_w, ops._p(self._qwt), self.k_pad,
                     self.ld_wt, None)
        # activations -> NHWC int8 (channel stride c_pad), pending_amax fused (layers.cpp:101)
        n, hh, ww, c = x.shape
        dev = x.z.device if fuse_in else x.device
        qa = torch.empty((n, hh, ww, self.c_pad), dtype=torch.int8, device=dev)
        pre = getattr(x, "_i8t_q", None) if not fuse_in else None
        if pre is not None and pre[0] is self:  # quantised by the producing block (i8t_bn_act_q)
            qa = pre[1]
        elif (not fuse_in and self.act_twin is not None and self.act_twin._qa_src is x and self.c_pad == c
              and self.act_twin._qa is not None and self.act_twin._qa.shape == qa.shape):
            # same input as the block's first conv (projection shortcut): its int8
            # tensor when the clips agree (they track the same tensor), else quantise
            tw = self.act_twin
            call("i8t_quantize_nearest_shared", h, ops._p(x), x.numel(), ops._p(qs.clip_a), ops._p(tw.qs.clip_a),
                 ops._p(tw._qa), ops._p(tw.qs.pending_amax) if ctx.track_amax else None, ops._p(qa),
                 ops._p(qs.pending_amax) if ctx.track_amax else None)
        elif fuse_in:  # BN-apply + ReLU + nearest quantise + amax in one pass over z
            bn = x.bn
            call("i8t_bn_act_quant", h, ops._p(x.z), n * hh * ww, c, ops._p(bn.stats), ops._p(bn.gamma),
                 ops._p(bn.beta), int(x.relu), ops._p(qs.clip_a), ops._p(qa),
                 ops._p(qs.pending_amax) if ctx.track_amax else None)
        else:
            call("i8t_quantize_nearest_rows", h, ops._p(x), n * hh * ww, c, ops._p(qs.clip_a), ops._p(qa),
                 self.c_pad, ops._p(qs.pending_amax) if ctx.track_amax else None, 1)
        self._qa = qa
        self._qa_src = x if (self.keep_qa_src and not fuse_in) else None
        z = torch.empty((n, p, q, self.out_c), dtype=torch.float32, device=dev)
        if self.depthwise:
            call("i8t_conv_dw_fwd", h, C.byref(g), ops._p(qa), self.c_pad, ops._p(self._qw), ops._p(qs.clip_a),
                 ops._p(qs.clip_w), ops._p(z), None)
        else:
            call("i8t_conv_fwd", h, C.byref(g), ops._p(qa), self.c_pad, ops._p(self._qw), self.ld_w,
                 ops._p(qs.clip_a), ops._p(qs.clip_w), ops._p(z), None)
        if TRACE is not None:
            TRACE(self, "fwd", x=None if fuse_in else x, qa=qa, qw=self._qw, z=z, w=self.weight)
        return z

    # -- backward (layers.cpp:113-126)
    def backward(self, gz, ctx: BackwardCtx):
        g = self._geom
        use_int8 = self.quantize_enabled and ctx.mode == Mode.INT8
        fuse_g = (isinstance(gz, BnGrad) and use_int8 and ctx.clip_search_enabled
                  and not self.qs.dsgc.due(ctx.iter) and gz.shape[-1] % 4 == 0)
        g_stats = None
        if (not fuse_g and isinstance(gz, BnGrad) and use_int8 and ctx.clip_search_enabled
                and self.qs.dsgc.due(ctx.iter) and gz.shape[-1] % 4 == 0 and BN_IMPL == "fused"):
            # a search step: the materialising BN backward also reduces the
            # search's first-pass statistics (max|g|, non-finite, sum g^2)
            g_stats = torch.empty(3, dtype=torch.float64, device=gz.g.device)
            gz = gz.materialize(stats=g_stats)
        elif not fuse_g:
            gz = dense_grad(gz)
            if use_int8 and ctx.clip_search_enabled and self.qs.dsgc.due(ctx.iter):
                g_stats = getattr(gz, "_i8t_stats", None)  # eager BN: reduced by its materialising pass
        if not use_int8:
            xc = self._x.permute(0, 3, 1, 2)
            gc = gz.permute(0, 3, 1, 2)
            groups = self.in_c if self.depthwise else 1
            with _fp32_exact():
                gi = torch.nn.grad.conv2d_input(xc.shape, self.weight, gc, (self.sh, self.sw), (self.ph, self.pw),
                                                groups=groups)
                self.grad_weight.copy_(torch.nn.grad.conv2d_weight(xc, self.weight.shape, gc, (self.sh, self.sw),
                                                                   (self.ph, self.pw), groups=groups))
            return gi.permute(0, 2, 3, 1).contiguous()
        h = ops.ctx()
        stream_in = ctx.grad_stream.clone() if TRACE is not None else None
        if fuse_g:  # BN backward computed on the fly inside the stochastic quantiser
            qg = quantize_gradient_bn_layer(self.qs, gz, ctx)
        else:
            gz = gz.contiguous()
            qg = quantize_gradient_layer(self.qs, gz, ctx, stats=g_stats)
        clip_g = self.qs.dsgc.clip_q_ptr()
        gdev = qg.device
        ga = torch.empty((g.n, g.h, g.w, g.c), dtype=torch.float32, device=gdev) if self.need_input_grad else None
        if self.depthwise:
            if self.need_input_grad:
                call("i8t_conv_dw_dgrad", h, C.byref(g), ops._p(qg), self.k_pad, ops._p(self._qw), ops._p(clip_g),
                     ops._p(self.qs.clip_w), ops._p(ga), None)
            if self.wgrad_acc is None:
                self.wgrad_acc = torch.empty((self.in_c, self.kh * self.kw), dtype=torch.int64, device=gdev)
            if ctx.wgrad_allreduce is None:
                call("i8t_conv_dw_wgrad", h, C.byref(g), ops._p(qg), ops._p(self._qa), self.c_pad, ops._p(clip_g),
                     ops._p(self.qs.clip_a), ops._p(self.wgrad_acc), ops._p(self.grad_weight))
            else:  # data parallel: exact int64 sum across ranks, rescaled after the allreduce
                call("i8t_conv_dw_wgrad", h, C.byref(g), ops._p(qg), ops._p(self._qa), self.c_pad, ops._p(clip_g),
                     ops._p(self.qs.clip_a), ops._p(self.wgrad_acc), None)
                acc, gw, clip_a, geo = self.wgrad_acc, self.grad_weight, self.qs.clip_a, g
                ctx.deferred.append((ctx.wgrad_allreduce(acc), lambda: call(
                    "i8t_conv_dw_wgrad_finalize", ops.ctx(), C.byref(geo), ops._p(acc), ops._p(clip_g), ops._p(clip_a),
                    ops._p(gw))))
        else:
            join, self.dgrad_join, self.join_done = self.dgrad_join, None, False
            if self.need_input_grad and join is not None and g.c % 4 == 0:
                add_g, add_y, add_bits = join
                if add_y is None and add_bits is None and add_g.is_contiguous() and add_g.shape == ga.shape:
                    # plain join (projection shortcut): accumulate into the addend in
                    # place -- a strided dgrad's tap-less phases then write nothing
                    ga = add_g
                if add_bits is not None:  # identity shortcut through the block ReLU, mask as packed bits
                    call("i8t_conv_dgrad_join_bits", h, C.byref(g), ops._p(qg), self.k_pad, ops._p(self._qwt),
                         self.ld_wt, ops._p(clip_g), ops._p(self.qs.clip_w), ops._p(ga), ops._p(add_g.contiguous()),
                         ops._p(add_bits))
                else:
                    call("i8t_conv_dgrad_join", h, C.byref(g), ops._p(qg), self.k_pad, ops._p(self._qwt), self.ld_wt,
                         ops._p(clip_g), ops._p(self.qs.clip_w), ops._p(ga), ops._p(add_g.contiguous()),
                         ops._p(add_y.contiguous() if add_y is not None else None))
                self.join_done = True
            elif self.need_input_grad:
                call("i8t_conv_dgrad", h, C.byref(g), ops._p(qg), self.k_pad, ops._p(self._qwt), self.ld_wt,
                     ops._p(clip_g), ops._p(self.qs.clip_w), ops._p(ga), None)
            if self.wgrad_acc is None and ctx.wgrad_allreduce is not None:
                self.wgrad_acc = torch.empty((self.kh * self.kw * self.c_pad, self.out_c), dtype=torch.int64,
                                             device=gdev)
            if ctx.wgrad_allreduce is None and ctx.wgrad_stream is not None:
                # the weight gradient on the side stream, after this layer's gradient quantiser
                side = ctx.wgrad_stream
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    call("i8t_conv_wgrad", ops.side_ctx(side), C.byref(g), ops._p(qg), self.k_pad, ops._p(self._qa),
                         self.c_pad, ops._p(clip_g), ops._p(self.qs.clip_a), None, ops._p(self.grad_weight), 1)
                qg.record_stream(side)
                self._qa.record_stream(side)
            elif ctx.wgrad_allreduce is None:  # single device: weights straight from the partials, no int64 copy
                call("i8t_conv_wgrad", h, C.byref(g), ops._p(qg), self.k_pad, ops._p(self._qa), self.c_pad,
                     ops._p(clip_g), ops._p(self.qs.clip_a), None, ops._p(self.grad_weight), 1)
            else:  # data parallel: exact int64 sum across ranks (async, overlapping the backward), then rescale
                call("i8t_conv_wgrad", h, C.byref(g), ops._p(qg), self.k_pad, ops._p(self._qa), self.c_pad,
                     ops._p(clip_g), ops._p(self.qs.clip_a), ops._p(self.wgrad_acc), None, 1)
                acc, gw, clip_a, geo, c_pad = self.wgrad_acc, self.grad_weight, self.qs.clip_a, g, self.c_pad
                ctx.deferred.append((ctx.wgrad_allreduce(acc), lambda: call(
                    "i8t_conv_wgrad_finalize", ops.ctx(), C.byref(geo), ops._p(acc), c_pad, ops._p(clip_g),
                    ops._p(clip_a), ops._p(gw), 1)))
        self._qa = None
        self._qg = qg if self.keep_qg else None
        if TRACE is not None:
            if ctx.wgrad_stream is not None:  # the instrumentation reads gw: wait for the side stream
                torch.cuda.current_stream().wait_stream(ctx.wgrad_stream)
            TRACE(self, "bwd", g=None if fuse_g else gz, qg=qg, stream_in=stream_in, stream_out=ctx.grad_stream,
                  ga=ga, gw=self.grad_weight if ctx.wgrad_allreduce is None else None)
        return ga


def quantize_gradient_layer(qs: QuantState, gz: torch.Tensor, ctx: BackwardCtx, stats=None) -> torch.Tensor:
    """quantize_gradient (layers.cpp:19-59) for an NHWC gradient [N,P,Q,K].
    stats: the search's first-pass statistics of gz when its producer reduced
    them (i8t_bn_bwd_apply_stats)."""
    n, p, q, k = gz.shape
    st = qs.dsgc
    st.period = ctx.clip_period
    due = st.due(ctx.iter) if ctx.clip_search_enabled else False
    qg = torch.empty(gz.shape, dtype=torch.int8, device=gz.device)
    if k % 4 == 0:
        n_img, ch, hw = n, k, p * q
    elif p * q == 1:  # fc gradient [N, K]: NCHW order == row-major order -> flat draw order
        n_img, ch, hw = 1, 1, n * k
    else:
        raise ValueError("quantize_gradient: conv output channels must be a multiple of 4")
    args = (ops.ctx(), st.ptr, ops._p(gz), n_img, ch, hw, ctx.iter, ctx.grid_resolution, ctx.refine_rounds,
            int(ctx.clip_search_enabled), int(due), int(ctx.lr_scaling_enabled), C.c_double(ctx.alpha),
            C.c_double(ctx.beta), ops.FORMS[ctx.form], ops._p(ctx.grad_stream), ops._p(qg), ch)
    if stats is not None and due:
        call("i8t_quantize_gradient_stats", *args, ops._p(stats))
    else:
        call("i8t_quantize_gradient", *args)
    if due or not ctx.clip_search_enabled:
        st.mark_searched(ctx.iter)
        st.clip_valid = True  # refreshed from the device view at step end (zero-gradient edge case)
    if k % 4:
        qg = torch.nn.functional.pad(qg, (0, ops.pad4(k) - k))  # channel stride k_pad for dgrad/wgrad
    return qg


def quantize_gradient_bn_layer(qs: QuantState, gz: "BnGrad", ctx: BackwardCtx) -> torch.Tensor:
    """quantize_gradient (layers.cpp:19-59) of a pending BN backward value on a
    non-search iteration: one pass reads (g, z) and writes the int8 gradient."""
    n, p, q, k = gz.shape
    st = qs.dsgc
    st.period = ctx.clip_period
    qg = torch.empty(gz.shape, dtype=torch.int8, device=gz.g.device)
    bn = gz.bn
    call("i8t_quantize_gradient_bn", ops.ctx(), st.ptr, ops._p(gz.g), ops._p(bn._z), n, k, p * q, ops._p(bn.stats),
         ops._p(bn.gamma), ops._p(bn.beta), gz.mode, ops._p(gz.mask_y), int(ctx.lr_scaling_enabled),
         C.c_double(ctx.alpha), C.c_double(ctx.beta), ops.FORMS[ctx.form], ops._p(ctx.grad_stream), ops._p(qg))
    return qg


class Dense(Layer):
    """INT8 fully connected layer (layers.hpp:117-139, layers.cpp:138-225):
    a 1x1 convolution over [N, 1, 1, in]; bias added in float; bias gradient
    = float(s_g * sum_i q_g[i, o]) (exact: every partial sum is a small
    integer multiple of s_g)."""
    kind = "fc"

    def __init__(self, in_f, out_f, gen=None, device="cuda"):
        self.conv = Conv2d(in_f, out_f, 1, 1, 0, False, gen, device)
        self.conv.weight = _kaiming((out_f, in_f, 1, 1), in_f, gen or torch.Generator().manual_seed(0), device)
        self.conv.grad_weight = torch.zeros_like(self.conv.weight)
        self.bias = torch.zeros(out_f, device=device)
        self.grad_bias = torch.zeros_like(self.bias)
        self.in_f, self.out_f = in_f, out_f
        self.qs = self.conv.qs
        self.conv.keep_qg = True

    @property
    def quantized(self):
        return self.conv.quantize_enabled

    def set_quantized(self, on):
        self.conv.set_quantized(on)

    def params(self):
        # [out, in] like the reference's Dense weight (layers.cpp:132): checkpoints interoperate
        return [ParamRef("weight", self.conv.weight.view(self.out_f, self.in_f),
                         self.conv.grad_weight.view(self.out_f, self.in_f)),
                ParamRef("bias", self.bias, self.grad_bias)]

    def param_attrs(self):
        return [(self.conv, "weight", "grad_weight"), (self, "bias", "grad_bias")]

    def forward(self, x, ctx):
        x = dense(x)
        self._in_shape = x.shape
        n = x.shape[0]
        z = self.conv.forward(x.reshape(n, 1, 1, self.in_f), ctx).reshape(n, self.out_f)
        return z + self.bias

    def backward(self, g, ctx):
        g = dense_grad(g)
        n = g.shape[0]
        g = g.contiguous()
        gi = self.conv.backward(g.reshape(n, 1, 1, self.out_f), ctx)
        if self.conv.quantize_enabled and ctx.mode == Mode.INT8:
            # sum_i s*q[i,o] in double == s * (integer sum) exactly (layers.cpp:214-220)
            sums = self.conv._qg.reshape(n, -1)[:, :self.out_f].sum(0, dtype=torch.int64)
            if ctx.wgrad_allreduce is not None:  # data parallel: the integer sums across ranks (exact)
                from . import dp
                dp.allreduce_int64_(sums)
            scale = self.qs.dsgc.buf[_SCALE_OFF:_SCALE_OFF + 4].view(torch.float32)
            self.grad_bias.copy_((sums.double() * scale.double()).float())
            self.conv._qg = None
        else:
            self.grad_bias.copy_(g.double().sum(0).float())
        return gi.reshape(self._in_shape)


class BatchNorm2d(Layer):
    """FP32 batch norm (layers.cpp:230-323).  Training: statistics and apply
    run in csrc/bnfuse.cu with the reference's double arithmetic; the forward
    returns a LazyAct and the backward a BnGrad so the neighbouring INT8
    convolutions fuse them into their quantisation passes."""
    kind = "bn"

    def __init__(self, c, momentum=0.1, eps=1e-5, device="cuda"):
        self.c = c
        self.gamma = torch.ones(c, device=device)
        self.beta = torch.zeros(c, device=device)
        self.grad_gamma = torch.zeros_like(self.gamma)
        self.grad_beta = torch.zeros_like(self.beta)
        self.running_mean = torch.zeros(c, device=device)
        self.running_var = torch.ones(c, device=device)
        self.momentum, self.eps = momentum, eps
        self.stats = torch.zeros(6 * c, dtype=torch.float64, device=device)  # mean, invstd, k*s1/m, k*s2/m, k = gamma*invstd, mask bounds
        self._z = None

    def params(self):
        return [ParamRef("gamma", self.gamma, self.grad_gamma), ParamRef("beta", self.beta, self.grad_beta)]

    def param_attrs(self):
        return [(self, "gamma", "grad_gamma"), (self, "beta", "grad_beta")]

    def buffers(self):
        return [ParamRef("running_mean", self.running_mean, None), ParamRef("running_var", self.running_var, None)]

    def _fusable(self, x):
        return BN_IMPL != "torch" and isinstance(x, torch.Tensor) and self.c % 4 == 0 and x.is_contiguous()

    def forward(self, x, ctx):
        x = dense(x)
        if not ctx.training:
            xc = x.permute(0, 3, 1, 2)
            y = F.batch_norm(xc, self.running_mean, self.running_var, self.gamma, self.beta, False, 0.0, self.eps)
            return y.permute(0, 2, 3, 1).contiguous()
        if self._fusable(x):
            n, h, w, c = x.shape
            call("i8t_bn_fwd_stats", ops.ctx(), ops._p(x), n * h * w, c, C.c_double(self.momentum),
                 C.c_double(self.eps), ops._p(self.stats), ops._p(self.running_mean), ops._p(self.running_var))
            self._z = x
            self._torch = False
            return LazyAct(x, self).materialize() if BN_IMPL == "eager" else LazyAct(x, self)
        xc = x.permute(0, 3, 1, 2)
        y, self._mean, self._invstd = torch.native_batch_norm(xc, self.gamma, self.beta, self.running_mean,
                                                              self.running_var, True, self.momentum, self.eps)
        self._x = xc
        self._torch = True
        return y.permute(0, 2, 3, 1).contiguous()

    def backward(self, g, ctx):
        if not self._torch:
            mode, mask_y = 0, None
            if isinstance(g, MaskedGrad):
                if g.mode == 1 and g.bn is not self:
                    g = g.materialize()
                else:
                    mode, mask_y, g = g.mode, g.mask_y, g.g
            if (isinstance(g, JoinGrad) and g.out is None and mode == 3 and JOIN_REDUCE and g.co_bn is not None
                    and g.co_bn is not self and not g.co_bn._torch and g.co_bn._z is not None
                    and g.co_bn._z.shape == self._z.shape):
                # the projection shortcut's BN on the same masked gradient, in the same pass
                n, h, w, c = g.shape
                co = g.co_bn
                out = torch.empty_like(g.gm)
                call("i8t_bn_bwd_reduce_join2", ops.ctx(), ops._p(g.gm), ops._p(g.g), ops._p(g.bits), ops._p(self._z),
                     n * h * w, c, ops._p(self.stats), ops._p(self.gamma), ops._p(self.beta), ops._p(mask_y),
                     ops._p(self.grad_gamma), ops._p(self.grad_beta), ops._p(co._z), ops._p(co.stats),
                     ops._p(co.gamma), ops._p(co.grad_gamma), ops._p(co.grad_beta), ops._p(out))
                co._reduced_for = out  # its own backward finds its sums done for this gradient
                g.out, g.gm, g.g, g.bits = out, None, None, None
                gb = BnGrad(out, self, mode, mask_y)
                if BN_IMPL == "eager":
                    stats = torch.empty(3, dtype=torch.float64, device=out.device)
                    res = gb.materialize(stats=stats)
                    res._i8t_stats = stats
                    return res
                return gb
            if isinstance(g, JoinGrad) and g.out is None and mode == 3 and JOIN_REDUCE:
                n, h, w, c = g.shape
                out = torch.empty_like(g.gm)
                call("i8t_bn_bwd_reduce_join", ops.ctx(), ops._p(g.gm), ops._p(g.g), ops._p(g.bits), ops._p(self._z),
                     n * h * w, c, ops._p(self.stats), ops._p(self.gamma), ops._p(self.beta), ops._p(mask_y),
                     ops._p(self.grad_gamma), ops._p(self.grad_beta), ops._p(out))
                g.out, g.gm, g.g, g.bits = out, None, None, None
                gb = BnGrad(out, self, mode, mask_y)
                if BN_IMPL == "eager":
                    stats = torch.empty(3, dtype=torch.float64, device=out.device)
                    res = gb.materialize(stats=stats)
                    res._i8t_stats = stats
                    return res
                return gb
            g = dense_grad(g).contiguous()
            n, h, w, c = g.shape
            if getattr(self, "_reduced_for", None) is g and mode == 3:
                self._reduced_for = None  # sums done in the main branch BN's pass (i8t_bn_bwd_reduce_join2)
            else:
                self._reduced_for = None
                call("i8t_bn_bwd_reduce", ops.ctx(), ops._p(g), ops._p(self._z), n * h * w, c, ops._p(self.stats),
                     ops._p(self.gamma), ops._p(self.beta), mode, ops._p(mask_y), ops._p(self.grad_gamma),
                     ops._p(self.grad_beta))
            gb = BnGrad(g, self, mode, mask_y)
            if BN_IMPL == "eager":  # the same kernel the fused path's search steps use, stats attached
                stats = torch.empty(3, dtype=torch.float64, device=g.device)
                out = gb.materialize(stats=stats)
                out._i8t_stats = stats
                return out
            return gb
        gc = dense_grad(g).contiguous().permute(0, 3, 1, 2)
        gi, gg, gb = torch.ops.aten.native_batch_norm_backward(gc, self._x, self.gamma, self.running_mean,
                                                               self.running_var, self._mean, self._invstd, True,
                                                               self.eps, [True, True, True])
        self.grad_gamma.copy_(gg)
        self.grad_beta.copy_(gb)
        self._x = None
        return gi.permute(0, 2, 3, 1).contiguous()


class ReLU(Layer):
    kind = "relu"

    def forward(self, x, ctx):
        if isinstance(x, LazyAct) and not x.relu:
            self._bn = x.bn  # mask recomputed from bn(z) in the backward (mask mode 1)
            return LazyAct(x.z, x.bn, relu=True)
        self._bn = None
        y = torch.relu(dense(x))
        if ctx.training:
            self._y = y
        return y

    def backward(self, g, ctx):
        g = dense_grad(g)
        if self._bn is not None:
            return MaskedGrad(g, 1, bn=self._bn)
        out = torch.where(self._y > 0, g, torch.zeros((), device=g.device, dtype=g.dtype))
        self._y = None
        return out


class MaxPool2d(Layer):
    """Max pooling with padding (EXT: the reference Pool2d has none, A.3-5) on
    csrc/pool.cu: the one-byte argmax replaces torch's int64 indices, and a
    preceding lazy BN + ReLU (the ResNet stem) is applied inside the pool so its
    fp32 output is never materialised."""
    kind = "maxpool"

    def __init__(self, k, s, p=0):
        self.k, self.s, self.p = k, s, p

    def forward(self, x, ctx):
        lazy = isinstance(x, LazyAct) and x.shape[-1] % 4 == 0
        src = x.z if lazy else dense(x).contiguous()
        n, h, w, c = src.shape
        if c % 4 or 2 * self.p > self.k:
            xc = src.permute(0, 3, 1, 2)
            y, self._idx = torch.ops.aten.max_pool2d_with_indices(xc, [self.k, self.k], [self.s, self.s],
                                                                  [self.p, self.p])
            self._xc, self._torch = xc, True
            return y.permute(0, 2, 3, 1).contiguous()
        P = (h + 2 * self.p - self.k) // self.s + 1
        Q = (w + 2 * self.p - self.k) // self.s + 1
        y = torch.empty((n, P, Q, c), dtype=torch.float32, device=src.device)
        idx = torch.empty((n, P, Q, c), dtype=torch.uint8, device=src.device)
        bn = x.bn if lazy else None
        call("i8t_maxpool_fwd", ops.ctx(), ops._p(src), n, h, w, c, self.k, self.s, self.p,
             ops._p(bn.stats) if bn else None, ops._p(bn.gamma) if bn else None, ops._p(bn.beta) if bn else None,
             int(x.relu) if lazy else 0, ops._p(y), ops._p(idx))
        self._torch = False
        if ctx.training:
            self._idx, self._in_shape = idx, (n, h, w, c)
        return y

    def backward(self, g, ctx):
        g = dense_grad(g).contiguous()
        if self._torch:
            gi = torch.ops.aten.max_pool2d_with_indices_backward(g.permute(0, 3, 1, 2), self._xc, [self.k, self.k],
                                                                 [self.s, self.s], [self.p, self.p], [1, 1], False,
                                                                 self._idx)
            self._xc = self._idx = None
            return gi.permute(0, 2, 3, 1).contiguous()
        n, h, w, c = self._in_shape
        gx = torch.empty((n, h, w, c), dtype=torch.float32, device=g.device)
        call("i8t_maxpool_bwd", ops.ctx(), ops._p(g), ops._p(self._idx), n, h, w, c, self.k, self.s, self.p,
             ops._p(gx))
        self._idx = None
        return gx


class AvgPool2d(Layer):
    """k x k average pooling, stride s, padding p (count_include_pad like torchvision)."""
    kind = "avgpool2d"

    def __init__(self, k, s, p=0):
        self.k, self.s, self.p = k, s, p

    def forward(self, x, ctx):
        x = dense(x)
        xc = x.permute(0, 3, 1, 2)
        self._xc = xc
        y = F.avg_pool2d(xc, self.k, self.s, self.p)
        return y.permute(0, 2, 3, 1).contiguous()

    def backward(self, g, ctx):
        g = dense_grad(g)
        gi = torch.ops.aten.avg_pool2d_backward(g.permute(0, 3, 1, 2), self._xc, [self.k, self.k], [self.s, self.s],
                                                [self.p, self.p], False, True, None)
        self._xc = None
        return gi.permute(0, 2, 3, 1).contiguous()


class Concat(Layer):
    """Parallel branches whose NHWC outputs are concatenated along channels
    (Inception blocks).  Backward splits the gradient per branch and runs the
    branches in forward order (the LCG stream is consumed in that order)."""
    kind = "concat"

    def __init__(self, branches):
        self.branches = list(branches)

    def forward(self, x, ctx):
        x = dense(x)
        outs = [dense(b.forward(x, ctx)) for b in self.branches]
        self._sizes = [o.shape[-1] for o in outs]
        return torch.cat(outs, dim=-1)

    def backward(self, g, ctx):
        parts = torch.split(dense_grad(g), self._sizes, dim=-1)
        gi = None
        for b, gp in zip(self.branches, parts):
            r = dense_grad(b.backward(gp.contiguous(), ctx))
            gi = r if gi is None else gi + r
        return gi

    def visit(self, prefix, fn):
        for i, b in enumerate(self.branches):
            b.visit(f"{prefix}/b{i}" if prefix else f"b{i}", fn)


class GlobalAvgPool(Layer):
    """Pool2d(kAvg) over the whole map (layers.cpp:383-388): the window sum is
    accumulated in double and divided once, float(sum / (h*w)), like the
    reference.  Its summation order differs from the reference's sequential
    one only in the last double bits (exact unless the window spans > 2^23 in
    magnitude), far below the final float rounding."""
    kind = "avgpool"

    def forward(self, x, ctx):
        x = dense(x).contiguous()
        self._shape = x.shape
        n, h, w, c = x.shape
        if x.is_cuda:
            y = torch.empty((n, c), dtype=torch.float32, device=x.device)
            call("i8t_global_avgpool_fwd", ops.ctx(), ops._p(x), n, h * w, c, ops._p(y))
            return y
        return (torch.sum(x, dim=(1, 2), dtype=torch.float64) / (h * w)).float()

    def backward(self, g, ctx):
        g = dense_grad(g).contiguous()
        n, h, w, c = self._shape
        if g.is_cuda and c % 4 == 0:
            gx = torch.empty((n, h, w, c), dtype=torch.float32, device=g.device)
            call("i8t_global_avgpool_bwd", ops.ctx(), ops._p(g), n, h * w, c, ops._p(gx))
            return gx
        return (g / (h * w)).reshape(n, 1, 1, c).expand(n, h, w, c).contiguous()


class Sequential(Layer):
    kind = "sequential"

    def __init__(self, children=None):
        self.children = list(children or [])

    def add(self, name, layer):
        self.children.append((name, layer))
        return layer

    def forward(self, x, ctx):
        for _, c in self.children:
            x = c.forward(x, ctx)
        return x

    def backward(self, g, ctx):
        for _, c in reversed(self.children):
            g = c.backward(g, ctx)
        return g

    def visit(self, prefix, fn):
        for name, c in self.children:
            c.visit(f"{prefix}/{name}" if prefix else name, fn)


class ResidualBlock(Layer):
    """relu(main(x) + shortcut(x)); backward runs main then shortcut
    (layers.cpp:451-464).  `main` is a BasicBlock (ResNet-20) or a Bottleneck
    (ResNet-50) Sequential."""
    kind = "resblock"

    def __init__(self, main: Sequential, shortcut: Sequential | None):
        self.main, self.shortcut, self.relu = main, shortcut, ReLU()
        self.next_conv = None  # first conv of the next block: its int8 input is written with the block output
        first = main.children[0][1] if main.children else None
        sc = shortcut.children[0][1] if shortcut and shortcut.children else None
        if isinstance(first, Conv2d) and isinstance(sc, Conv2d) and SHARE_ACT:
            sc.act_twin = first  # both quantise the block input x
            first.keep_qa_src = True

    def forward(self, x, ctx):
        x = dense(x)
        y = self.main.forward(x, ctx)
        sc = self.shortcut.forward(x, ctx) if self.shortcut else x
        first = self.main.children[0][1] if self.main.children else None
        if isinstance(first, Conv2d):
            first._qa_src = None  # the shortcut has taken its int8 input (or not): drop the reference
        if isinstance(y, LazyAct) and not y.relu:  # relu(bn3(z3) + shortcut) in one pass
            bits = None
            if ctx.training and y.z.numel() % 4 == 0:  # the backward keeps one bit of y per element
                bits = torch.empty(((y.z.numel() + 31) // 32,), dtype=torch.int32, device=y.z.device)
            out = LazyAct(y.z, y.bn, relu=True).materialize(res=sc, quant_for=self.next_conv, ctx=ctx,
                                                            mask_bits=bits)
            self._bits, self._fused = bits, True
            self._y = out if bits is None else None
            return out
        self._fused = False
        return self.relu.forward(dense(y) + dense(sc), ctx)

    def backward(self, g, ctx):
        jg = g if isinstance(g, JoinGrad) and self._fused and self._bits is not None else None
        g = jg if jg is not None else dense_grad(g)
        if jg is not None and self.shortcut and self.shortcut.children and JOIN_REDUCE2:
            last = self.shortcut.children[-1][1]
            if isinstance(last, BatchNorm2d):
                jg.co_bn = last  # the shortcut BN's sums ride along with the main branch's last BN
        if self._fused:
            gl = MaskedGrad(g, 3, mask_y=self._bits) if self._bits is not None else MaskedGrad(g, 2, mask_y=self._y)
            first = self.main.children[0][1] if self.main.children else None
            joinable = isinstance(first, Conv2d) and not first.depthwise and JOIN_FUSION
            if joinable and not self.shortcut:  # identity: conv1's dgrad adds g * (y > 0)
                first.dgrad_join = (g, self._y, self._bits)
            gm = dense_grad(self.main.backward(gl, ctx))
            if jg is not None:  # the main branch's last BN materialised the incoming join (or does it now)
                g = jg.materialize()
            if joinable and not self.shortcut and first.join_done:
                return gm
            if self.shortcut:
                sc = self.shortcut.children[0][1] if self.shortcut.children else None
                sc_join = isinstance(sc, Conv2d) and not sc.depthwise and JOIN_PROJ
                if sc_join:  # projection: the downsample conv's dgrad adds the main-branch gradient
                    sc.dgrad_join = (gm, None, None)
                gs = dense_grad(self.shortcut.backward(gl, ctx))
                if sc_join and sc.join_done:
                    return gs
                return gm + gs
            if self._bits is not None and JOIN_REDUCE and BN_IMPL == "fused":
                jout = JoinGrad(gm, g, self._bits)
                self._bits = self._y = None
                return jout
            out = torch.empty_like(gm)
            if self._bits is not None:
                call("i8t_add_masked_bits", ops.ctx(), ops._p(gm), ops._p(g), ops._p(self._bits), gm.numel(),
                     ops._p(out))
            else:
                call("i8t_add_masked", ops.ctx(), ops._p(gm), ops._p(g), ops._p(self._y), gm.numel(), ops._p(out))
            self._bits = self._y = None
            return out
        g = self.relu.backward(g, ctx)
        gm = dense_grad(self.main.backward(g, ctx))
        gs = dense_grad(self.shortcut.backward(g, ctx)) if self.shortcut else g
        return gm + gs

    def visit(self, prefix, fn):
        self.main.visit(prefix, fn)
        if self.shortcut:
            self.shortcut.visit(prefix, fn)


class InvertedResidual(Layer):
    """MobileNetV2 block (layers.cpp:466-502): 1x1 expand, 3x3 depthwise, 1x1
    project; skip when stride 1 and in == out."""
    kind = "invres"

    def __init__(self, body: Sequential, use_skip: bool):
        self.body, self.use_skip = body, use_skip

    def forward(self, x, ctx):
        x = dense(x)
        y = self.body.forward(x, ctx)
        if self.use_skip:
            return y.materialize(res=x) if isinstance(y, LazyAct) else y + x
        return y

    def backward(self, g, ctx):
        g = dense_grad(g)
        gb = dense_grad(self.body.backward(g, ctx))
        return gb + g if self.use_skip else gb

    def visit(self, prefix, fn):
        self.body.visit(prefix, fn)


class SoftmaxCrossEntropy:
    """Mean softmax cross-entropy in double (layers.cpp:507-529); returns the
    loss as a 0-d CUDA double tensor and g_logits = float((p - y) / N)."""

    @staticmethod
    def loss_and_grad(logits: torch.Tensor, labels: torch.Tensor, total_n: int | None = None, bad=None):
        """total_n: the global batch under data parallelism (default: local).
        bad: optional int32 [1] device tensor that receives the divergence flag
        (non-finite loss or logits) of the same pass."""
        n = logits.shape[0] if total_n is None else total_n
        if logits.is_cuda and labels.dtype == torch.int64:
            logits = logits.contiguous()
            g = torch.empty_like(logits)
            loss = torch.empty((), dtype=torch.float64, device=logits.device)
            flag = bad if bad is not None else torch.empty(1, dtype=torch.int32, device=logits.device)
            call("i8t_softmax_ce", ops.ctx(), ops._p(logits), ops._p(labels.contiguous()), logits.shape[0],
                 logits.shape[1], n, ops._p(g), ops._p(loss), ops._p(flag))
            return loss, g
        if bad is not None:
            bad.copy_(((~torch.isfinite(logits).all())).to(torch.int32).reshape(1))
        ld = logits.double()
        logz = torch.logsumexp(ld, dim=1)
        loss = (logz - ld.gather(1, labels.view(-1, 1)).squeeze(1)).sum() / n
        p = torch.exp(ld - logz.view(-1, 1))
        p[torch.arange(logits.shape[0], device=logits.device), labels] -= 1.0
        if bad is not None:
            bad.bitwise_or_((~torch.isfinite(loss)).to(torch.int32).reshape(1))
        return loss, (p / n).float()


def int8_replace(root: Layer) -> int:
    """Figure-6 replacement (layers.cpp:536-546): flip every conv / conv_dw / fc to INT8."""
    count = 0

    def fn(_, layer):
        nonlocal count
        if layer.kind in ("conv", "conv_dw", "fc"):
            layer.set_quantized(True)
            count += 1
    root.visit("", fn)
    return count


def leaves(root: Layer):
    out = []
    root.visit("", lambda path, layer: out.append((path, layer)))
    return out
