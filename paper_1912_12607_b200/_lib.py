"""ctypes binding of libi8t_cuda.so, generated from include/i8t_cuda.h.

The prototypes are parsed from the header itself so the Python side can never
drift from the C-ABI.  There is no fallback: if the library or a CUDA device
is missing, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
HEADER = os.path.join(ROOT, "include", "i8t_cuda.h")
LIB_PATH = os.path.join(PKG, "libi8t_cuda.so")

I8T_OK, I8T_EINVAL, I8T_EDOMAIN, I8T_ECUDA, I8T_EUNSUPPORTED = range(5)


class ConvGeom(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n", "c", "h", "w", "k", "kh", "kw",
                                        "stride_h", "stride_w", "pad_h", "pad_w")] + \
               [("depthwise", C.c_int32), ("floor_mode", C.c_int32)]

    def out_hw(self):
        return ((self.h + 2 * self.pad_h - self.kh) // self.stride_h + 1,
                (self.w + 2 * self.pad_w - self.kw) // self.stride_w + 1)


class WqDesc(C.Structure):
    """i8t_wq_desc (include/i8t_cuda.h)."""
    _fields_ = [("w", C.c_void_p), ("clip", C.c_void_p), ("q_krsc", C.c_void_p), ("q_crsk", C.c_void_p)] + \
               [(n, C.c_int32) for n in ("k", "c", "rs", "c_pad", "ld_krsc", "k_pad", "ld_crsk", "src_krsc")]


class DsgcView(C.Structure):
    _fields_ = [("clip", C.c_float), ("scale", C.c_float), ("max_abs", C.c_float), ("flags", C.c_uint32),
                ("last_dc", C.c_double), ("lr_scale", C.c_double), ("eps_norm", C.c_double),
                ("ghat_sqnorm", C.c_double), ("iter_of_last_update", C.c_int64), ("period", C.c_int64),
                ("clip_q", C.c_float), ("reserved", C.c_uint32)]


_CTYPES = {
    "int": C.c_int, "int32_t": C.c_int32, "int64_t": C.c_int64, "uint32_t": C.c_uint32,
    "uint64_t": C.c_uint64, "double": C.c_double, "float": C.c_float, "void": None,
    "const char*": C.c_char_p,
}


def _ptype(decl: str):
    d = " ".join(decl.replace("const ", "").split())
    d = d.rsplit(" ", 1)[0] if not d.endswith("*") and " " in d else d
    if "i8t_conv_geom" in d:
        return C.POINTER(ConvGeom)
    if "i8t_dsgc_view" in d:
        return C.POINTER(DsgcView)
    if "i8t_allreduce_fn" in d:
        return C.c_void_p
    if "i8t_ctx**" in d.replace(" ", ""):
        return C.POINTER(C.c_void_p)
    if "*" in d:
        return C.c_void_p
    return _CTYPES[d.strip()]


def parse_header(path: str = HEADER) -> dict[str, tuple]:
    """{name: (restype, [argtypes])} for every i8t_* function declared."""
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"\b(int|int64_t|uint64_t|const char\*)\s+(i8t_\w+)\s*\(([^)]*)\)\s*;", src):
        ret, name, args = m.group(1), m.group(2), m.group(3).strip()
        argtypes = [] if args in ("", "void") else [_ptype(a.strip()) for a in args.split(",")]
        out[name] = (_CTYPES[ret], argtypes)
    return out


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in parse_header().items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class I8tError(RuntimeError):
    pass


def check(rc: int, what: str = ""):
    if rc == I8T_OK:
        return
    msg = lib().i8t_last_error().decode()
    if rc == I8T_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == I8T_EDOMAIN:
        raise ArithmeticError(f"{what}: {msg}")
    raise I8tError(f"{what}: status {rc}: {msg}")


def _arg(a):
    # device tensors are passed by their data pointer; the caller's argument
    # tuple owns them until the call (and the launch it enqueues) has returned
    return C.c_void_p(a.data_ptr()) if hasattr(a, "data_ptr") else a


def call(name: str, *args):
    check(getattr(lib(), name)(*(_arg(a) for a in args)), name)
