"""Torch-facing mirror of the reference operator API (namespace i8t,
proj/core/include/i8t/*.hpp), running every op through the C-ABI of
libi8t_cuda.so on the current CUDA stream.

Names and argument meaning follow the reference: ``quantize``,
``dequantize``, ``quantize_partitioned``, ``max_abs``, ``sq_l2_norm``,
``dot``, ``has_nonfinite``, ``gemm_i8``, ``conv2d_q``, ``conv2d_backward_q``,
``cosine_distance``, ``measure_dc``, ``search_clip``, ``maybe_update``,
``scale_factor``, ``effective_lr``.  Errors map like the reference's
exceptions: ValueError <- std::invalid_argument, ArithmeticError <-
std::domain_error.  Tensors are torch CUDA tensors; layouts are the
reference's (NCHW / KCRS) at this API, converted on the device to the
kernels' NHWC / KRSC / CRSK layouts.  There is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import ConvGeom, DsgcView, I8tError, call, lib  # noqa: F401 (I8tError re-exported)

# --------------------------------------------------------------------------- context
_ctx = {}


def ctx(stream: torch.cuda.Stream | None = None) -> C.c_void_p:
    """One i8t_ctx per device, bound to the current torch stream."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1912_12607_b200 needs a CUDA device (no CPU fallback)")
    dev = torch.cuda.current_device()
    s = (stream or torch.cuda.current_stream()).cuda_stream
    h = _ctx.get(dev)
    if h is None:
        h = C.c_void_p()
        call("i8t_ctx_create", C.c_void_p(s), C.byref(h))
        _ctx[dev] = h
    else:
        call("i8t_ctx_set_stream", h, C.c_void_p(s))
    return h


_side_ctx: dict = {}


def side_ctx(stream: torch.cuda.Stream) -> C.c_void_p:
    """A second i8t_ctx per device (its own scratch) for work on a side stream
    that overlaps the main context's (the weight gradients)."""
    dev = torch.cuda.current_device()
    h = _side_ctx.get(dev)
    if h is None:
        h = C.c_void_p()
        call("i8t_ctx_create", C.c_void_p(stream.cuda_stream), C.byref(h))
        _side_ctx[dev] = h
    else:
        call("i8t_ctx_set_stream", h, C.c_void_p(stream.cuda_stream))
    return h


def check():
    """Synchronise and raise the latched device error (reference exceptions)."""
    call("i8t_ctx_check", ctx())


def launch_count() -> int:
    return int(lib().i8t_launch_count())


def _p(t: torch.Tensor | None):
    """A device-pointer argument of `call`: the tensor itself (None = NULL).
    `call` converts it to its data pointer while its own argument tuple keeps
    the tensor alive, so temporaries created inline (``_p(_dev_f32(clip))``)
    live until the launch they feed has been enqueued; the stream-ordered
    caching allocator makes any later reuse safe."""
    return t


def _dev_f32(v, device=None) -> torch.Tensor:
    if isinstance(v, torch.Tensor):
        return v.reshape(1).to(torch.float32)
    return torch.tensor([float(v)], dtype=torch.float32, device=device or "cuda")


def quant_scale(clip: float) -> float:
    """QuantParams::from_clip (quantize.cpp:11-14): s = float(c / 127.0f)."""
    c = torch.tensor(clip, dtype=torch.float32)
    if not (c > 0 and torch.isfinite(c)):
        raise ValueError("QuantParams: clip must be positive and finite")
    return float(c / torch.tensor(127.0, dtype=torch.float32))


def _check_clip(clip):
    if not isinstance(clip, torch.Tensor):
        quant_scale(clip)


@dataclass
class QuantizedTensor:
    """QuantizedTensor (quantize.hpp:20-26): int8 payload + clip/scale."""
    q: torch.Tensor
    clip: float
    shape: tuple = field(default=())

    @property
    def scale(self) -> float:
        return quant_scale(self.clip)


# --------------------------------------------------------------------------- quantizers
def quantize(x: torch.Tensor, clip, stochastic: bool = False, stream_state: torch.Tensor | None = None,
             amax: torch.Tensor | None = None, accumulate_amax: bool = False) -> torch.Tensor:
    """quantize(x, from_clip(clip), mode, stream) (quantize.cpp:33-43), flat order.
    stream_state: int32 CUDA tensor [1] holding the LcgStream state (advanced in place)."""
    if stochastic != (stream_state is not None):
        raise ValueError("quantize: stream required iff mode is stochastic")
    _check_clip(clip)
    x = x.contiguous()
    q = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    d_clip = _dev_f32(clip, x.device)
    h = ctx()
    if stochastic:  # any length: the library pads a ragged tail and rewinds the stream over it
        call("i8t_quantize_stochastic", h, _p(x), x.numel(), _p(d_clip), _p(stream_state), _p(q))
    else:
        call("i8t_quantize_nearest", h, _p(x), x.numel(), _p(d_clip), _p(q), _p(amax), int(accumulate_amax))
    return q


def quantize_partitioned(x: torch.Tensor, clip, base_seed: int, partitions: int) -> torch.Tensor:
    """quantize_partitioned (quantize.cpp:45-79)."""
    if partitions < 1:
        raise ValueError("quantize_partitioned: partitions must be >= 1")
    _check_clip(clip)
    x = x.contiguous()
    q = torch.empty(x.shape, dtype=torch.int8, device=x.device)
    call("i8t_quantize_partitioned", ctx(), _p(x), x.numel(), _p(_dev_f32(clip, x.device)),
         C.c_uint32(base_seed & 0xFFFFFFFF), partitions, _p(q))
    return q


def dequantize(q: torch.Tensor, clip) -> torch.Tensor:
    """dequantize (quantize.cpp:81-87): float(q) * scale."""
    out = torch.empty(q.shape, dtype=torch.float32, device=q.device)
    call("i8t_dequantize", ctx(), _p(q.contiguous()), q.numel(), _p(_dev_f32(clip, q.device)), _p(out))
    return out


def quantize_act_nhwc(x_nchw: torch.Tensor, clip, c_pad: int | None = None, amax=None, accumulate_amax=False):
    """NCHW float -> NHWC int8 with channel stride c_pad (the conv kernels' A layout)."""
    n, c, h, w = x_nchw.shape
    c_pad = c_pad or pad4(c)
    q = torch.empty((n, h, w, c_pad), dtype=torch.int8, device=x_nchw.device)
    call("i8t_quantize_nearest_nchw_to_nhwc", ctx(), _p(x_nchw.contiguous()), n, c, h * w,
         _p(_dev_f32(clip, x_nchw.device)), _p(q), c_pad, _p(amax), int(accumulate_amax))
    return q


def pad4(c: int) -> int:
    return (c + 3) // 4 * 4


def pad16(c: int) -> int:
    return (c + 15) // 16 * 16


def quantize_weight(w: torch.Tensor, clip, krsc_src: bool = False, c_pad=None, k_pad=None, amax=None):
    """Weights (KCRS float) -> (KRSC int8 [K][ld], CRSK int8 [C][ld]) nearest."""
    k, c, kh, kw = (w.shape[0], w.shape[3], w.shape[1], w.shape[2]) if krsc_src else w.shape
    c_pad = c_pad or pad4(c)
    k_pad = k_pad or pad4(k)
    ld1, ld2 = pad16(kh * kw * c_pad), pad16(kh * kw * k_pad)
    q1 = torch.empty((k, ld1), dtype=torch.int8, device=w.device)
    q2 = torch.empty((c, ld2), dtype=torch.int8, device=w.device)
    call("i8t_quantize_weight", ctx(), _p(w.contiguous()), int(krsc_src), k, c, kh, kw, _p(_dev_f32(clip, w.device)),
         _p(q1), c_pad, ld1, _p(q2), k_pad, ld2, _p(amax))
    return q1, q2


def nchw_to_nhwc_i8(q: torch.Tensor, c_pad: int | None = None) -> torch.Tensor:
    n, c, h, w = q.shape
    c_pad = c_pad or pad4(c)
    out = torch.empty((n, h, w, c_pad), dtype=torch.int8, device=q.device)
    call("i8t_nchw_to_nhwc_i8", ctx(), _p(q.contiguous()), n, c, h * w, _p(out), c_pad)
    return out


def kcrs_to_krsc_i8(q: torch.Tensor, c_pad=None):
    k, c, kh, kw = q.shape
    c_pad = c_pad or pad4(c)
    ld = pad16(kh * kw * c_pad)
    out = torch.empty((k, ld), dtype=torch.int8, device=q.device)
    call("i8t_kcrs_to_krsc_i8", ctx(), _p(q.contiguous()), k, c, kh, kw, _p(out), c_pad, ld)
    return out, ld


def kcrs_to_crsk_i8(q: torch.Tensor, k_pad=None):
    k, c, kh, kw = q.shape
    k_pad = k_pad or pad4(k)
    ld = pad16(kh * kw * k_pad)
    out = torch.empty((c, ld), dtype=torch.int8, device=q.device)
    call("i8t_kcrs_to_crsk_i8", ctx(), _p(q.contiguous()), k, c, kh, kw, _p(out), k_pad, ld)
    return out, ld


def nhwc_to_nchw(x: torch.Tensor, c: int) -> torch.Tensor:
    """float NHWC [N,H,W,ld] -> NCHW [N,c,H,W]."""
    n, h, w, ld = x.shape
    out = torch.empty((n, c, h, w), dtype=torch.float32, device=x.device)
    call("i8t_nhwc_to_nchw_f32", ctx(), _p(x.contiguous()), n, c, h * w, ld, _p(out))
    return out


# --------------------------------------------------------------------------- reductions
def max_abs(x: torch.Tensor) -> float:
    out = torch.empty(1, dtype=torch.float32, device=x.device)
    call("i8t_max_abs", ctx(), _p(x.contiguous()), x.numel(), _p(out))
    return float(out.item())


def sq_l2_norm(x: torch.Tensor) -> float:
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    call("i8t_sq_l2_norm", ctx(), _p(x.contiguous()), x.numel(), _p(out))
    return float(out.item())


def dot(a: torch.Tensor, b: torch.Tensor) -> float:
    if a.numel() != b.numel():
        raise ValueError("dot: size mismatch")
    out = torch.empty(1, dtype=torch.float64, device=a.device)
    call("i8t_dot", ctx(), _p(a.contiguous()), _p(b.contiguous()), a.numel(), _p(out))
    return float(out.item())


def has_nonfinite(x: torch.Tensor) -> bool:
    out = torch.empty(1, dtype=torch.int32, device=x.device)
    call("i8t_has_nonfinite", ctx(), _p(x.contiguous()), x.numel(), _p(out))
    return bool(out.item())


# --------------------------------------------------------------------------- DSGC / DCLR
def cosine_distance(g: torch.Tensor, h: torch.Tensor) -> float:
    """cosine_distance (clip.cpp:8-22)."""
    if g.shape != h.shape:
        raise ValueError("cosine_distance: shape mismatch")
    out = torch.empty(1, dtype=torch.float64, device=g.device)
    call("i8t_cosine_distance", ctx(), _p(g.contiguous()), _p(h.contiguous()), g.numel(), _p(out))
    return float(out.item())


def measure_dc(g: torch.Tensor, clip: float) -> float:
    """measure_dc (clip.cpp:24-28)."""
    out = torch.empty(1, dtype=torch.float64, device=g.device)
    call("i8t_measure_dc", ctx(), _p(g.contiguous()), g.numel(), C.c_float(clip), _p(out))
    check()
    return float(out.item())


def search_clip(g: torch.Tensor, grid_resolution: int = 32, refine_rounds: int = 2, prev_clip: float = 0.0):
    """search_clip (clip.cpp:30-78) -> (clip, dc)."""
    c = torch.empty(1, dtype=torch.float32, device=g.device)
    d = torch.empty(1, dtype=torch.float64, device=g.device)
    call("i8t_search_clip", ctx(), _p(g.contiguous()), g.numel(), grid_resolution, refine_rounds,
         C.c_float(prev_clip), _p(c), _p(d))
    check()
    return float(c.item()), float(d.item())


FORMS = {"exp": 0, "exponential": 0, "linear": 1, "quadratic": 2}


def scale_factor(dc: float, alpha: float = 20.0, beta: float = 0.1, form: str = "exp") -> float:
    """scale_factor (lr_scale.cpp:8-20)."""
    out = C.c_double()
    call("i8t_scale_factor", C.c_double(dc), C.c_double(alpha), C.c_double(beta), FORMS[form], C.byref(out))
    return out.value


def effective_lr(base_lr: float, dc_per_layer: dict, alpha=20.0, beta=0.1, form="exp") -> dict:
    """effective_lr (lr_scale.cpp:22-29)."""
    if not base_lr > 0.0:
        raise ValueError("effective_lr: base_lr must be > 0")
    return {k: base_lr * scale_factor(v, alpha, beta, form) for k, v in sorted(dc_per_layer.items())}


class DsgcState:
    """Device-resident ClipState + QuantState measurements of one layer
    (clip.hpp:12-18, layers.hpp:28-38), with the host mirror needed to decide
    Periodic-Update due-ness without a device round trip."""

    def __init__(self, period: int = 100, layer_id: str = "", device=None):
        size = int(lib().i8t_dsgc_state_size())
        self.buf = torch.zeros(size, dtype=torch.uint8, device=device or "cuda")
        self.layer_id = layer_id
        self.period = period
        call("i8t_dsgc_init", ctx(), _p(self.buf), period)
        self.iter_of_last_update = -1
        self.clip_valid = False  # host mirror of clip > 0 (refreshed by sync())

    @property
    def ptr(self):
        return _p(self.buf)

    def view(self) -> DsgcView:
        v = DsgcView()
        call("i8t_dsgc_read", ctx(), self.ptr, C.byref(v))
        return v

    def write(self, v: DsgcView):
        call("i8t_dsgc_write", ctx(), self.ptr, C.byref(v))
        self.sync(v)

    def sync(self, v: DsgcView | None = None):
        v = v or self.view()
        self.clip_valid = v.clip > 0.0
        self.iter_of_last_update = v.iter_of_last_update
        return v

    def due(self, it: int) -> bool:
        """maybe_update's condition (clip.cpp:82-84)."""
        if it < self.iter_of_last_update:
            raise ValueError("maybe_update: iter went backwards")
        return (not self.clip_valid) or self.iter_of_last_update < 0 or (it - self.iter_of_last_update) >= self.period

    def mark_searched(self, it: int):
        self.iter_of_last_update = it


def maybe_update(state: DsgcState, g: torch.Tensor, it: int, grid_resolution=32, refine_rounds=2):
    """maybe_update (clip.cpp:80-93) on a device state."""
    if grid_resolution < 8:
        raise ValueError("search_clip: grid resolution must be >= 8")
    due = state.due(it)
    call("i8t_maybe_update", ctx(), state.ptr, _p(g.contiguous()), g.numel(), it, grid_resolution, refine_rounds,
         int(due))
    check()
    return state.sync()


def new_lcg_state(seed: int, device=None) -> torch.Tensor:
    """Device copy of LcgStream(seed) state (quantize.hpp:36)."""
    return torch.tensor([C.c_int32(seed & 0xFFFFFFFF).value], dtype=torch.int32, device=device or "cuda")


def lcg_value(state: torch.Tensor) -> int:
    return int(state.item()) & 0xFFFFFFFF


def quantize_gradient(state: DsgcState, g: torch.Tensor, it: int, lcg_state: torch.Tensor, *, nhwc: bool = False,
                      grid_resolution=32, refine_rounds=2, search_enabled=True, lr_scaling_enabled=True,
                      alpha=20.0, beta=0.1, form="exp", out: torch.Tensor | None = None) -> torch.Tensor:
    """quantize_gradient (layers.cpp:19-59), fused on the device.

    g: NCHW tensor (nhwc=False, flat draw order) or a channels-last NHWC
    buffer [N,H,W,C] (nhwc=True) whose draw order is still the reference's
    NCHW order.  Returns the int8 gradient in g's physical layout.  The scale,
    d_c, phi, eps and g_hat^2 stay on the device in `state` (state.view())."""
    g = g.contiguous()
    if nhwc:
        n, h, w, c = g.shape
        n_img, ch, hw = n, c, h * w
    else:
        n_img, ch, hw = 1, 1, g.numel()
    due = state.due(it) if search_enabled else False
    q = out if out is not None else torch.empty(g.shape, dtype=torch.int8, device=g.device)
    call("i8t_quantize_gradient", ctx(), state.ptr, _p(g), n_img, ch, hw, it, grid_resolution, refine_rounds,
         int(search_enabled), int(due), int(lr_scaling_enabled), C.c_double(alpha), C.c_double(beta),
         FORMS[form], _p(lcg_state), _p(q), ch)
    if search_enabled and due:
        state.mark_searched(it)
    if not search_enabled:
        state.iter_of_last_update = it
    return q


def sgd_dclr_(w: torch.Tensor, grad: torch.Tensor, base_lr: float, state: DsgcState | None = None):
    """Trainer::train_step update (train.cpp:97-117): w -= float(lr * g)."""
    call("i8t_sgd_dclr", ctx(), _p(w), _p(grad.contiguous()), w.numel(), C.c_double(base_lr),
         state.ptr if state is not None else None, None)


# --------------------------------------------------------------------------- GEMM / conv
def gemm_i8(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """gemm_i8 (gemm.cpp:18-40): exact int32 C = A . B."""
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError("gemm_i8: inner dimensions do not match")
    if k > 130000:
        raise ValueError("gemm_i8: depth exceeds i32 overflow bound")
    c = torch.empty((m, n), dtype=torch.int32, device=a.device)
    call("i8t_gemm_s8", ctx(), _p(a.contiguous()), _p(b.contiguous()), m, k, n, _p(c))
    return c


def gemm_i8_fused_lhs(a: torch.Tensor, clip, stochastic: bool, stream_state: torch.Tensor | None,
                      b: torch.Tensor) -> torch.Tensor:
    """gemm_i8_fused_lhs (gemm.cpp:49-64): C = quantize(A fp32, from_clip(clip), mode[, stream]) . B,
    quantised on the device into the GEMM's operand; bit-identical to quantize() + gemm_i8()
    incl. the stream state (advanced by m*k when stochastic)."""
    if stochastic != (stream_state is not None):
        raise ValueError("quantize: stream required iff mode is stochastic")
    if a.dim() != 2:
        raise ValueError("gemm_i8_fused_lhs: lhs must be 2-D")
    _check_clip(clip)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise ValueError("gemm_i8: inner dimensions do not match")
    c = torch.empty((m, n), dtype=torch.int32, device=a.device)
    call("i8t_gemm_s8_fused_lhs", ctx(), _p(a.contiguous().float()), m, k, _p(_dev_f32(clip, a.device)),
         int(stochastic), _p(stream_state), _p(b.contiguous()), n, _p(c))
    return c


def im2col_i8(x: torch.Tensor, g: ConvGeom, channel: int | None = None) -> torch.Tensor:
    """im2col_i8 / im2col_channel_i8 (conv.cpp:23-47, 98-106): NCHW int8 ->
    col [C*kh*kw (or kh*kw), N*P*Q] int8, zero padding."""
    p, q = g.out_hw()
    c_lo, c_hi = (0, g.c) if channel is None else (channel, channel + 1)
    col = torch.empty(((c_hi - c_lo) * g.kh * g.kw, g.n * p * q), dtype=torch.int8, device=x.device)
    call("i8t_im2col_s8", ctx(), _p(x.contiguous()), C.byref(g), c_lo, c_hi, _p(col))
    return col


def geom(n, c, h, w, k, kh, kw=None, stride=1, pad=0, depthwise=False, floor_mode=True, stride_w=None,
         pad_w=None) -> ConvGeom:
    kw = kh if kw is None else kw
    return ConvGeom(n, c, h, w, k, kh, kw, stride, stride if stride_w is None else stride_w, pad,
                    pad if pad_w is None else pad_w, int(depthwise), int(floor_mode))


def conv_fwd_nhwc(g: ConvGeom, qa_nhwc, c_pad, qw_krsc, ld_w, clip_a, clip_w, want_acc=False, z_out=None):
    """tcgen05 forward conv on kernel layouts; returns (z NHWC [NPQ,K] float, acc int32 or None)."""
    p, q = g.out_hw()
    z = z_out if z_out is not None else torch.empty((g.n * p * q, g.k), dtype=torch.float32, device=qa_nhwc.device)
    acc = torch.empty((g.n * p * q, g.k), dtype=torch.int32, device=qa_nhwc.device) if want_acc else None
    call("i8t_conv_fwd", ctx(), C.byref(g), _p(qa_nhwc), c_pad, _p(qw_krsc), ld_w, _p(_dev_f32(clip_a)),
         _p(_dev_f32(clip_w)), _p(z), _p(acc))
    return z, acc


def conv_dgrad_nhwc(g: ConvGeom, qg_nhwc, k_pad, qw_crsk, ld_wt, clip_g, clip_w, want_acc=False, out=None):
    ga = out if out is not None else torch.empty((g.n * g.h * g.w, g.c), dtype=torch.float32, device=qg_nhwc.device)
    acc = torch.empty((g.n * g.h * g.w, g.c), dtype=torch.int32, device=qg_nhwc.device) if want_acc else None
    call("i8t_conv_dgrad", ctx(), C.byref(g), _p(qg_nhwc), k_pad, _p(qw_crsk), ld_wt, _p(_dev_f32(clip_g)),
         _p(_dev_f32(clip_w)), _p(ga), _p(acc))
    return ga, acc


def conv_wgrad_nhwc(g: ConvGeom, qg_nhwc, k_pad, qa_nhwc, c_pad, clip_g, clip_a, out_kcrs=True, acc=None, gw=None):
    rows = g.kh * g.kw * c_pad
    acc = acc if acc is not None else torch.empty((rows, g.k), dtype=torch.int64, device=qg_nhwc.device)
    if gw is None:
        shape = (g.k, g.c, g.kh, g.kw) if out_kcrs else (g.k, g.kh, g.kw, g.c)
        gw = torch.empty(shape, dtype=torch.float32, device=qg_nhwc.device)
    call("i8t_conv_wgrad", ctx(), C.byref(g), _p(qg_nhwc), k_pad, _p(qa_nhwc), c_pad, _p(_dev_f32(clip_g)),
         _p(_dev_f32(clip_a)), _p(acc), _p(gw), int(out_kcrs))
    return gw, acc


def conv2d_q(qa: torch.Tensor, clip_a: float, qw: torch.Tensor, clip_w: float, g: ConvGeom, want_acc=False):
    """conv2d_q (conv.cpp:108-145): NCHW int8 a, KCRS int8 w -> NCHW float z
    (and the NKPQ int32 accumulator when want_acc)."""
    _check_clip(clip_a)
    _check_clip(clip_w)
    p, q = g.out_hw()
    if g.depthwise:
        c_pad = g.c
        a_n = nchw_to_nhwc_i8(qa, c_pad)
        z = torch.empty((g.n * p * q, g.c), dtype=torch.float32, device=qa.device)
        acc = torch.empty((g.n * p * q, g.c), dtype=torch.int32, device=qa.device) if want_acc else None
        call("i8t_conv_dw_fwd", ctx(), C.byref(g), _p(a_n), c_pad, _p(qw.contiguous()), _p(_dev_f32(clip_a)),
             _p(_dev_f32(clip_w)), _p(z), _p(acc))
        kout = g.c
    else:
        c_pad = pad4(g.c)
        a_n = nchw_to_nhwc_i8(qa, c_pad)
        w_n, ld = kcrs_to_krsc_i8(qw, c_pad)
        z, acc = conv_fwd_nhwc(g, a_n, c_pad, w_n, ld, clip_a, clip_w, want_acc)
        kout = g.k
    zc = nhwc_to_nchw(z.view(g.n, p, q, kout), kout)
    if want_acc:
        return zc, acc.view(g.n, p, q, kout).permute(0, 3, 1, 2).contiguous()
    return zc


def conv2d_backward_q(qg: torch.Tensor, clip_g: float, qa: torch.Tensor, clip_a: float, qw: torch.Tensor,
                      clip_w: float, g: ConvGeom, want_acc=False):
    """conv2d_backward_q (conv.cpp:147-205) -> (gW KCRS float, gA NCHW float)
    [+ (wgrad int64 acc KCRS, dgrad int32 acc NCHW) when want_acc]."""
    for c in (clip_g, clip_a, clip_w):
        _check_clip(c)
    p, q = g.out_hw()
    if g.depthwise:
        c_pad = g.c
        g_n = nchw_to_nhwc_i8(qg, c_pad)
        a_n = nchw_to_nhwc_i8(qa, c_pad)
        ga = torch.empty((g.n * g.h * g.w, g.c), dtype=torch.float32, device=qg.device)
        acc_a = torch.empty((g.n * g.h * g.w, g.c), dtype=torch.int32, device=qg.device) if want_acc else None
        call("i8t_conv_dw_dgrad", ctx(), C.byref(g), _p(g_n), c_pad, _p(qw.contiguous()), _p(_dev_f32(clip_g)),
             _p(_dev_f32(clip_w)), _p(ga), _p(acc_a))
        acc_w = torch.empty((g.c, g.kh * g.kw), dtype=torch.int64, device=qg.device)
        gw = torch.empty((g.c, 1, g.kh, g.kw), dtype=torch.float32, device=qg.device)
        call("i8t_conv_dw_wgrad", ctx(), C.byref(g), _p(g_n), _p(a_n), c_pad, _p(_dev_f32(clip_g)),
             _p(_dev_f32(clip_a)), _p(acc_w), _p(gw))
        gac = nhwc_to_nchw(ga.view(g.n, g.h, g.w, g.c), g.c)
        if want_acc:
            return gw, gac, acc_w.view(g.c, 1, g.kh, g.kw), acc_a.view(g.n, g.h, g.w, g.c).permute(0, 3, 1, 2).contiguous()
        return gw, gac
    c_pad, k_pad = pad4(g.c), pad4(g.k)
    g_n = nchw_to_nhwc_i8(qg, k_pad)
    a_n = nchw_to_nhwc_i8(qa, c_pad)
    wt, ldt = kcrs_to_crsk_i8(qw, k_pad)
    ga, acc_a = conv_dgrad_nhwc(g, g_n, k_pad, wt, ldt, clip_g, clip_w, want_acc)
    gw, acc_w = conv_wgrad_nhwc(g, g_n, k_pad, a_n, c_pad, clip_g, clip_a, out_kcrs=True)
    gac = nhwc_to_nchw(ga.view(g.n, g.h, g.w, g.c), g.c)
    if want_acc:
        accw = acc_w.view(g.kh, g.kw, c_pad, g.k)[:, :, :g.c, :].permute(3, 2, 0, 1).contiguous()
        return gw, gac, accw, acc_a.view(g.n, g.h, g.w, g.c).permute(0, 3, 1, 2).contiguous()
    return gw, gac
