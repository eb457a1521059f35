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
        VP = C.c_void_p
        L.ref_model_new.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.c_int, C.POINTER(VP)]
        L.ref_model_free.argtypes = [VP]
        L.ref_model_free.restype = None
        L.ref_model_ntensors.argtypes = [VP]
        L.ref_model_tensor_info.argtypes = [VP, C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int), P_I64]
        L.ref_model_tensor_get.argtypes = [VP, C.c_int, P_F32]
        L.ref_model_tensor_set.argtypes = [VP, C.c_int, P_F32]
        L.ref_model_int8_replace.argtypes = [VP]
        L.ref_trainer_new.argtypes = [VP, P_F64, P_I64, C.POINTER(VP)]
        L.ref_trainer_free.argtypes = [VP]
        L.ref_trainer_free.restype = None
        L.ref_trainer_calibrate.argtypes = [VP, VP, P_F32, C.c_int64]
        L.ref_trainer_finish_calibration.argtypes = [VP]
        L.ref_trainer_refresh.argtypes = [VP]
        L.ref_train_step.argtypes = [VP, VP, P_F32, C.c_int64, np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS"),
                                     C.c_int64, C.c_int64, P_F64, P_F64]
        L.ref_trainer_quant_state.argtypes = [VP, C.c_int, P_F32, C.POINTER(ClipState)]
        L.ref_save_checkpoint.argtypes = [VP, C.c_char_p]
        L.ref_load_checkpoint.argtypes = [VP, C.c_char_p]
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


# ---------------------------------------------------------------- Model / Trainer / checkpoint (train.cpp)
FORMS = {"exp": 0, "linear": 1, "quadratic": 2}


class RefModel:
    """A reference Model (models.cpp, or the probe's res_s1 / mbv2_s1)."""

    def __init__(self, name, seed=1, side=32, classes=10):
        self.h = C.c_void_p()
        _check(lib().ref_model_new(name.encode(), seed, side, classes, C.byref(self.h)))
        self.name, self.side, self.classes = name, side, classes

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_model_free(self.h)

    def tensors(self) -> dict:
        out = {}
        L = lib()
        for i in range(L.ref_model_ntensors(self.h)):
            nb = C.create_string_buffer(256)
            rank = C.c_int()
            dims = np.zeros(8, np.int64)
            _check(L.ref_model_tensor_info(self.h, i, nb, 256, C.byref(rank), dims))
            t = np.empty(tuple(int(d) for d in dims[:rank.value]), np.float32)
            _check(L.ref_model_tensor_get(self.h, i, t.reshape(-1)))
            out[nb.value.decode()] = t
        return out

    def set_tensors(self, values: dict):
        L = lib()
        names = list(self.tensors().keys())
        for i, name in enumerate(names):
            if name in values:
                _check(L.ref_model_tensor_set(self.h, i, f32(values[name]).reshape(-1)))

    def int8_replace(self) -> int:
        return lib().ref_model_int8_replace(self.h)

    def save(self, path):
        _check(lib().ref_save_checkpoint(self.h, path.encode()))

    def load(self, path):
        rc = lib().ref_load_checkpoint(self.h, path.encode())
        if rc:
            raise RuntimeError("reference load_checkpoint failed")


class RefTrainer:
    """The reference Trainer (train.cpp:12-120) on a RefModel."""

    def __init__(self, model: RefModel, base_lr=0.1, momentum=0.0, alpha=20.0, beta=0.1, mode="int8",
                 schedule="cosine", lr_scaling=True, clip_enabled=True, clip_period=100, seed=1, grid=32, rounds=2,
                 form="exp"):
        self.model = model
        self.h = C.c_void_p()
        cfg = np.array([base_lr, momentum, alpha, beta], np.float64)
        icfg = np.array([int(mode == "int8"), int(schedule == "constant"), int(lr_scaling), int(clip_enabled),
                         clip_period, seed, grid, rounds, FORMS[form]], np.int64)
        _check(lib().ref_trainer_new(model.h, cfg, icfg, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_trainer_free(self.h)

    def calibrate(self, images):
        _check(lib().ref_trainer_calibrate(self.h, self.model.h, f32(images).reshape(-1), images.shape[0]))

    def finish_calibration(self):
        _check(lib().ref_trainer_finish_calibration(self.h))

    def refresh_wa_clips(self):
        _check(lib().ref_trainer_refresh(self.h))

    def train_step(self, images, labels, it, total, n_quant):
        out = np.zeros(3, np.float64)
        st = np.zeros(5 * max(n_quant, 1), np.float64)
        _check(lib().ref_train_step(self.h, self.model.h, f32(images).reshape(-1), images.shape[0],
                                    np.ascontiguousarray(labels, np.int32), it, total, out, st))
        return dict(loss=out[0], diverged=bool(out[1]), base_lr_t=out[2], layers=st.reshape(-1, 5)[:n_quant])

    def quant_state(self, i):
        f = np.zeros(3, np.float32)
        cs = ClipState()
        _check(lib().ref_trainer_quant_state(self.h, i, f, C.byref(cs)))
        return f, cs
