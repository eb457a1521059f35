"""ctypes bindings of oracle/liboracle.so (the C restatement) -- TEST ONLY.

numpy in, numpy out.  Every wrapper raises ValueError for OR_EINVAL (the
reference's std::invalid_argument) and ArithmeticError for OR_EDOMAIN (the
reference's std::domain_error).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_lib = None

P_F32 = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
P_I8 = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
P_I32 = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
P_I64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


class Geom(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n", "c", "h", "w", "k", "kh", "kw",
                                        "stride_h", "stride_w", "pad_h", "pad_w")] + \
               [("depthwise", C.c_int32), ("floor_mode", C.c_int32)]


class ClipState(C.Structure):
    _fields_ = [("clip", C.c_float), ("last_dc", C.c_double),
                ("iter_of_last_update", C.c_int64), ("period", C.c_int64)]


def build():
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.or_lcg_next.argtypes = [C.POINTER(C.c_uint32)]
        L.or_lcg_next.restype = C.c_uint32
        L.or_lcg_jump.argtypes = [C.c_uint32, C.c_uint64]
        L.or_lcg_jump.restype = C.c_uint32
        L.or_quant_params.argtypes = [C.c_float, C.POINTER(C.c_float)]
        L.or_quantize.argtypes = [P_F32, C.c_int64, C.c_float, C.c_int, C.POINTER(C.c_uint32), P_I8]
        L.or_quantize_partitioned.argtypes = [P_F32, C.c_int64, C.c_float, C.c_uint32, C.c_int, P_I8]
        L.or_dequantize.argtypes = [P_I8, C.c_int64, C.c_float, P_F32]
        L.or_dequantize.restype = None
        L.or_sq_l2_norm.argtypes = [P_F32, C.c_int64]
        L.or_sq_l2_norm.restype = C.c_double
        L.or_dot.argtypes = [P_F32, P_F32, C.c_int64]
        L.or_dot.restype = C.c_double
        L.or_max_abs.argtypes = [P_F32, C.c_int64]
        L.or_max_abs.restype = C.c_float
        L.or_has_nonfinite.argtypes = [P_F32, C.c_int64]
        L.or_gemm_i8.argtypes = [P_I8, P_I8, C.c_int64, C.c_int64, C.c_int64, P_I32]
        L.or_gemm_i8.restype = None
        L.or_geom_validate.argtypes = [C.POINTER(Geom)]
        L.or_out_h.argtypes = [C.POINTER(Geom)]
        L.or_out_h.restype = C.c_int64
        L.or_out_w.argtypes = [C.POINTER(Geom)]
        L.or_out_w.restype = C.c_int64
        L.or_im2col_i8.argtypes = [P_I8, C.POINTER(Geom), P_I8]
        L.or_conv_fwd.argtypes = [P_I8, P_I8, C.POINTER(Geom), C.c_float, C.c_float, P_I32, P_F32]
        L.or_conv_dgrad.argtypes = [P_I8, P_I8, C.POINTER(Geom), C.c_float, C.c_float, P_I64, P_F32]
        L.or_conv_wgrad.argtypes = [P_I8, P_I8, C.POINTER(Geom), C.c_float, C.c_float, P_I64, P_F32]
        L.or_cosine_distance.argtypes = [P_F32, P_F32, C.c_int64]
        L.or_cosine_distance.restype = C.c_double
        L.or_measure_dc.argtypes = [P_F32, C.c_int64, C.c_float, C.POINTER(C.c_double)]
        L.or_search_clip.argtypes = [P_F32, C.c_int64, C.c_int, C.c_int, C.c_float,
                                     C.POINTER(C.c_float), C.POINTER(C.c_double)]
        L.or_maybe_update.argtypes = [C.POINTER(ClipState), P_F32, C.c_int64, C.c_int64, C.c_int, C.c_int]
        L.or_scale_factor.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.or_quantize_gradient.argtypes = [
            C.POINTER(ClipState), P_F32, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
            C.c_double, C.c_double, C.c_int, C.POINTER(C.c_uint32), P_I8, C.POINTER(C.c_float),
            np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
        L.or_sgd_update.argtypes = [P_F32, P_F32, C.c_int64, C.c_double]
        L.or_sgd_update.restype = None
        L.or_fill_gaussian.argtypes = [P_F32, C.c_int64, C.c_uint64, C.c_double, C.c_int]
        L.or_fill_gaussian.restype = None
        L.or_fill_gradient_like.argtypes = [P_F32, C.c_int64, C.c_uint64, C.c_double, C.c_double]
        L.or_fill_gradient_like.restype = None
        P_F64 = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        L.or_bn_forward_train.argtypes = [P_F32, C.c_int64, C.c_int64, C.c_int64, P_F32, P_F32, P_F32, P_F32,
                                          C.c_double, C.c_double, P_F32, P_F32, P_F64]
        L.or_bn_forward_train.restype = None
        L.or_bn_forward_eval.argtypes = [P_F32, C.c_int64, C.c_int64, C.c_int64, P_F32, P_F32, P_F32, P_F32,
                                         C.c_double, P_F32]
        L.or_bn_forward_eval.restype = None
        L.or_bn_backward.argtypes = [P_F32, P_F32, P_F64, C.c_int64, C.c_int64, C.c_int64, P_F32, P_F32, P_F32,
                                     P_F32]
        L.or_bn_backward.restype = None
        L.or_pool_forward.argtypes = [P_F32] + [C.c_int64] * 4 + [C.c_int] + [C.c_int64] * 3 + [P_F32, C.c_void_p]
        L.or_pool_backward.argtypes = [P_F32, C.c_void_p] + [C.c_int64] * 4 + [C.c_int] + [C.c_int64] * 3 + [P_F32]
        L.or_softmax_ce.argtypes = [P_F32, C.c_int64, C.c_int64, np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                    P_F32, C.POINTER(C.c_int)]
        L.or_softmax_ce.restype = C.c_double
        L.or_sgd_momentum_update.argtypes = [P_F32, P_F32, P_F32, C.c_int64, C.c_double, C.c_double]
        L.or_sgd_momentum_update.restype = None
        L.or_conv_fwd_f32.argtypes = [P_F32, P_F32, C.POINTER(Geom), P_F32]
        _lib = L
    return _lib


def _check(rc):
    if rc == 1:
        raise ValueError("oracle: invalid argument")
    if rc == 2:
        raise ArithmeticError("oracle: non-finite input")
    if rc != 0:
        raise RuntimeError(f"oracle: status {rc}")


def f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


# ---------------------------------------------------------------- LCG / quantizer
def lcg_next(state: int) -> tuple[int, int]:
    s = C.c_uint32(state)
    v = lib().or_lcg_next(C.byref(s))
    return v, s.value


def lcg_jump(state: int, k: int) -> int:
    return lib().or_lcg_jump(state, k)


def quant_scale(clip: float) -> float:
    s = C.c_float()
    _check(lib().or_quant_params(clip, C.byref(s)))
    return s.value


def quantize(x, clip, stochastic=False, stream=None):
    """Returns (q int8, new_stream_state or None)."""
    x = f32(x)
    q = np.empty(x.shape, np.int8)
    if stochastic:
        s = C.c_uint32(stream)
        _check(lib().or_quantize(x.ravel(), x.size, clip, 1, C.byref(s), q.reshape(-1)))
        return q, s.value
    _check(lib().or_quantize(x.ravel(), x.size, clip, 0, None, q.reshape(-1)))
    return q, None


def quantize_partitioned(x, clip, base_seed, partitions):
    x = f32(x)
    q = np.empty(x.shape, np.int8)
    _check(lib().or_quantize_partitioned(x.ravel(), x.size, clip, base_seed, partitions, q.reshape(-1)))
    return q


def dequantize(q, scale):
    q = np.ascontiguousarray(q, np.int8)
    out = np.empty(q.shape, np.float32)
    lib().or_dequantize(q.ravel(), q.size, scale, out.reshape(-1))
    return out


def max_abs(x):
    x = f32(x)
    return lib().or_max_abs(x.ravel(), x.size)


def sq_l2_norm(x):
    x = f32(x)
    return lib().or_sq_l2_norm(x.ravel(), x.size)


def dot(a, b):
    a, b = f32(a), f32(b)
    return lib().or_dot(a.ravel(), b.ravel(), a.size)


def has_nonfinite(x):
    x = f32(x)
    return bool(lib().or_has_nonfinite(x.ravel(), x.size))


def gemm_i8(a, b):
    a = np.ascontiguousarray(a, np.int8)
    b = np.ascontiguousarray(b, np.int8)
    m, k = a.shape
    k2, n = b.shape
    assert k == k2
    c = np.empty((m, n), np.int32)
    lib().or_gemm_i8(a, b, m, k, n, c)
    return c


# ---------------------------------------------------------------- convolution
def geom(n, c, h, w, k, kh, kw, stride=1, pad=0, depthwise=False, floor_mode=True,
         stride_w=None, pad_w=None) -> Geom:
    return Geom(n, c, h, w, k, kh, kw, stride, stride if stride_w is None else stride_w,
                pad, pad if pad_w is None else pad_w, int(depthwise), int(floor_mode))


def out_hw(g: Geom):
    _check(lib().or_geom_validate(C.byref(g)))
    return lib().or_out_h(C.byref(g)), lib().or_out_w(C.byref(g))


def weight_shape(g: Geom):
    return (g.c, 1, g.kh, g.kw) if g.depthwise else (g.k, g.c, g.kh, g.kw)


def output_shape(g: Geom):
    p, q = out_hw(g)
    return (g.n, g.c if g.depthwise else g.k, p, q)


def im2col_i8(x, g: Geom):
    p, q = out_hw(g)
    out = np.empty((g.c * g.kh * g.kw, g.n * p * q), np.int8)
    _check(lib().or_im2col_i8(np.ascontiguousarray(x, np.int8).ravel(), C.byref(g), out))
    return out


def conv_fwd(qa, qw, g: Geom, s_a, s_w):
    """Returns (acc int32 NKPQ, z float32 NKPQ)."""
    shp = output_shape(g)
    acc = np.empty(shp, np.int32)
    z = np.empty(shp, np.float32)
    _check(lib().or_conv_fwd(np.ascontiguousarray(qa, np.int8).ravel(), np.ascontiguousarray(qw, np.int8).ravel(),
                             C.byref(g), s_a, s_w, acc.reshape(-1), z.reshape(-1)))
    return acc, z


def conv_dgrad(qg, qw, g: Geom, s_g, s_w):
    """Returns (acc int64 NCHW, ga float32 NCHW)."""
    shp = (g.n, g.c, g.h, g.w)
    acc = np.empty(shp, np.int64)
    ga = np.empty(shp, np.float32)
    _check(lib().or_conv_dgrad(np.ascontiguousarray(qg, np.int8).ravel(), np.ascontiguousarray(qw, np.int8).ravel(),
                               C.byref(g), s_g, s_w, acc.reshape(-1), ga.reshape(-1)))
    return acc, ga


def conv_wgrad(qg, qa, g: Geom, s_g, s_a):
    """Returns (acc int64 weight-shape, gw float32)."""
    shp = weight_shape(g)
    acc = np.empty(shp, np.int64)
    gw = np.empty(shp, np.float32)
    _check(lib().or_conv_wgrad(np.ascontiguousarray(qg, np.int8).ravel(), np.ascontiguousarray(qa, np.int8).ravel(),
                               C.byref(g), s_g, s_a, acc.reshape(-1), gw.reshape(-1)))
    return acc, gw


# ---------------------------------------------------------------- DSGC / DCLR
def cosine_distance(g, h):
    g, h = f32(g), f32(h)
    return lib().or_cosine_distance(g.ravel(), h.ravel(), g.size)


def measure_dc(g, clip):
    g = f32(g)
    d = C.c_double()
    _check(lib().or_measure_dc(g.ravel(), g.size, clip, C.byref(d)))
    return d.value


def search_clip(g, grid=32, rounds=2, prev_clip=0.0):
    g = f32(g)
    c, d = C.c_float(), C.c_double()
    _check(lib().or_search_clip(g.ravel(), g.size, grid, rounds, prev_clip, C.byref(c), C.byref(d)))
    return c.value, d.value


def new_clip_state(period=100) -> ClipState:
    return ClipState(0.0, 0.0, -1, period)


def maybe_update(st: ClipState, g, it, grid=32, rounds=2):
    g = f32(g)
    _check(lib().or_maybe_update(C.byref(st), g.ravel(), g.size, it, grid, rounds))
    return st


FORMS = {"exp": 0, "linear": 1, "quadratic": 2}


def scale_factor(dc, alpha=20.0, beta=0.1, form="exp"):
    out = C.c_double()
    _check(lib().or_scale_factor(dc, alpha, beta, FORMS[form], C.byref(out)))
    return out.value


def quantize_gradient(st: ClipState, g, it, stream, grid=32, rounds=2, search=True, lr_scaling=True,
                      alpha=20.0, beta=0.1, form="exp"):
    """layers.cpp:19-59.  Returns (q, scale, stream_after, stats{dc,lr_scale,eps_norm,ghat_sqnorm})."""
    g = f32(g)
    q = np.empty(g.shape, np.int8)
    s = C.c_uint32(stream)
    sc = C.c_float()
    stats = np.zeros(4, np.float64)
    _check(lib().or_quantize_gradient(C.byref(st), g.ravel(), g.size, it, grid, rounds, int(search),
                                      int(lr_scaling), alpha, beta, FORMS[form], C.byref(s), q.reshape(-1),
                                      C.byref(sc), stats))
    return q, sc.value, s.value, dict(dc=stats[0], lr_scale=stats[1], eps_norm=stats[2], ghat_sqnorm=stats[3])


def sgd_update(w, g, lr):
    w = f32(w).copy()
    lib().or_sgd_update(w.reshape(-1), f32(g).reshape(-1), w.size, lr)
    return w


# ---------------------------------------------------------------- synthetic inputs
def gaussian(shape, seed, stddev=1.0, relu=False):
    x = np.empty(shape, np.float32)
    lib().or_fill_gaussian(x.reshape(-1), x.size, seed, stddev, int(relu))
    return x


def gradient_like(shape, seed, scale=1e-4, outlier_rate=0.01):
    x = np.empty(shape, np.float32)
    lib().or_fill_gradient_like(x.reshape(-1), x.size, seed, scale, outlier_rate)
    return x
