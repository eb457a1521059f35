"""ctypes bindings of oracle/_ref/libi8t_ref.so -- the UNMODIFIED reference
compiled from /root/reference sources by oracle/Makefile.  TEST / BASELINE ONLY.

``available()`` is False where the .so was never built (it is built here in
the dev container and travels to the GPU box as a prebuilt file).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .lib import P_F32, P_I8, P_I32, ClipState, _check, f32

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libi8t_ref.so")
REF_SRC = "/root/reference/proj/core"
_lib = None
P_I64 = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
P_F64 = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> bool:
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
    return os.path.exists(LIB_PATH)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.ref_lcg_next.argtypes = [C.POINTER(C.c_uint32)]
        L.ref_lcg_next.restype = C.c_uint32
        L.ref_lcg_uniform.argtypes = [C.POINTER(C.c_uint32)]
        L.ref_lcg_uniform.restype = C.c_double
        L.ref_quant_params.argtypes = [C.c_float, C.POINTER(C.c_float)]
        L.ref_quantize.argtypes = [P_F32, C.c_int64, C.c_float, C.c_int, C.POINTER(C.c_uint32), P_I8]
        L.ref_quantize_partitioned.argtypes = [P_F32, C.c_int64, C.c_float, C.c_uint32, C.c_int, C.c_int, P_I8]
        L.ref_dequantize.argtypes = [P_I8, C.c_int64, C.c_float, P_F32]
        L.ref_max_abs.argtypes = [P_F32, C.c_int64]
        L.ref_max_abs.restype = C.c_float
        L.ref_sq_l2_norm.argtypes = [P_F32, C.c_int64]
        L.ref_sq_l2_norm.restype = C.c_double
        L.ref_dot.argtypes = [P_F32, P_F32, C.c_int64]
        L.ref_dot.restype = C.c_double
        L.ref_has_nonfinite.argtypes = [P_F32, C.c_int64]
        L.ref_gemm_i8.argtypes = [P_I8, P_I8, C.c_int64, C.c_int64, C.c_int64, C.c_int, P_I32]
        L.ref_im2col_i8.argtypes = [P_I8, P_I64, P_I8]
        L.ref_conv2d_q.argtypes = [P_I8, C.c_float, P_I8, C.c_float, P_I64, C.c_int, P_F32]
        L.ref_conv2d_backward_q.argtypes = [P_I8, C.c_float, P_I8, C.c_float, P_I8, C.c_float, P_I64, C.c_int,
                                            P_F32, P_F32]
        L.ref_cosine_distance.argtypes = [P_F32, P_F32, C.c_int64]
        L.ref_cosine_distance.restype = C.c_double
        L.ref_measure_dc.argtypes = [P_F32, C.c_int64, C.c_float, C.POINTER(C.c_double)]
        L.ref_search_clip.argtypes = [P_F32, C.c_int64, C.c_int, C.c_int, C.c_float, C.POINTER(C.c_float),
                                      C.POINTER(C.c_double)]
        L.ref_maybe_update.argtypes = [C.POINTER(ClipState), P_F32, C.c_int64, C.c_int64, C.c_int, C.c_int]
        L.ref_scale_factor.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_double)]
        L.ref_conv_layer_step.argtypes = [P_I64, P_F32, P_F32, P_F32, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                          C.POINTER(C.c_uint32), C.POINTER(ClipState), P_F32, P_F32, P_F32, P_F64]
        L.ref_fill_gaussian.argtypes = [P_F32, C.c_int64, C.c_uint64, C.c_double]
        L.ref_fill_gaussian.restype = None
        _lib = L
    return _lib


def gvec(n, c, h, w, k, kh, kw, stride=1, pad=0, depthwise=False):
    return np.array([n, c, h, w, k, kh, kw, stride, pad, int(depthwise)], np.int64)


def out_shape(gv):
    n, c, h, w, k, kh, kw, s, p, dw = (int(v) for v in gv)
    return (n, c if dw else k, (h + 2 * p - kh) // s + 1, (w + 2 * p - kw) // s + 1)


def w_shape(gv):
    n, c, h, w, k, kh, kw, s, p, dw = (int(v) for v in gv)
    return (c, 1, kh, kw) if dw else (k, c, kh, kw)


def quantize(x, clip, stochastic=False, stream=None):
    x = f32(x)
    q = np.empty(x.shape, np.int8)
    if stochastic:
        s = C.c_uint32(stream)
        _check(lib().ref_quantize(x.ravel(), x.size, clip, 1, C.byref(s), q.reshape(-1)))
        return q, s.value
    _check(lib().ref_quantize(x.ravel(), x.size, clip, 0, None, q.reshape(-1)))
    return q, None


def quantize_partitioned(x, clip, seed, parts, threads=1):
    x = f32(x)
    q = np.empty(x.shape, np.int8)
    _check(lib().ref_quantize_partitioned(x.ravel(), x.size, clip, seed, parts, threads, q.reshape(-1)))
    return q


def conv2d_q(qa, clip_a, qw, clip_w, gv, threads=1):
    z = np.empty(out_shape(gv), np.float32)
    _check(lib().ref_conv2d_q(np.ascontiguousarray(qa, np.int8).ravel(), clip_a,
                              np.ascontiguousarray(qw, np.int8).ravel(), clip_w, gv, threads, z.reshape(-1)))
    return z


def conv2d_backward_q(qg, clip_g, qa, clip_a, qw, clip_w, gv, threads=1):
    gw = np.empty(w_shape(gv), np.float32)
    n, c, h, w = (int(v) for v in gv[:4])
    ga = np.empty((n, c, h, w), np.float32)
    _check(lib().ref_conv2d_backward_q(np.ascontiguousarray(qg, np.int8).ravel(), clip_g,
                                       np.ascontiguousarray(qa, np.int8).ravel(), clip_a,
                                       np.ascontiguousarray(qw, np.int8).ravel(), clip_w, gv, threads,
                                       gw.reshape(-1), ga.reshape(-1)))
    return gw, ga


def measure_dc(g, clip):
    g = f32(g)
    d = C.c_double()
    _check(lib().ref_measure_dc(g.ravel(), g.size, clip, C.byref(d)))
    return d.value


def search_clip(g, grid=32, rounds=2, prev_clip=0.0):
    g = f32(g)
    c, d = C.c_float(), C.c_double()
    _check(lib().ref_search_clip(g.ravel(), g.size, grid, rounds, prev_clip, C.byref(c), C.byref(d)))
    return c.value, d.value


def maybe_update(st: ClipState, g, it, grid=32, rounds=2):
    g = f32(g)
    _check(lib().ref_maybe_update(C.byref(st), g.ravel(), g.size, it, grid, rounds))
    return st


def scale_factor(dc, alpha=20.0, beta=0.1, form=0):
    out = C.c_double()
    _check(lib().ref_scale_factor(dc, alpha, beta, form, C.byref(out)))
    return out.value


def conv_layer_step(gv, weight, x, g_out, it, stream, cs: ClipState, period=100, grid=32, rounds=2):
    """Reference Conv2d INT8 forward+backward (layers.cpp:98-126).  Returns
    (z, gw, ga, stream_after, stats[clip_w, clip_a, grad_clip, dc, lr_scale, eps, ghat_sq])."""
    z = np.empty(out_shape(gv), np.float32)
    gw = np.empty(w_shape(gv), np.float32)
    ga = np.empty(tuple(int(v) for v in gv[:4]), np.float32)
    stats = np.zeros(7, np.float64)
    s = C.c_uint32(stream)
    _check(lib().ref_conv_layer_step(gv, f32(weight).ravel(), f32(x).ravel(), f32(g_out).ravel(), it, period,
                                     grid, rounds, C.byref(s), C.byref(cs), z.reshape(-1), gw.reshape(-1),
                                     ga.reshape(-1), stats))
    return z, gw, ga, s.value, stats
