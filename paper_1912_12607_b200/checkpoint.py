"""Checkpoint and trace I/O for the trainer.

* I8FT container (checkpoint.hpp:9-15): magic "I8FT", u32 version,
  u32 n_tensors, u32 n_clip; tensor records (name, rank, u32 dims, f32
  payload) for every parameter and buffer of every leaf, sorted by name;
  clip records (name, f32 clip, f64 last_dc, i64 iter_of_last_update, i64
  period, f32 clip_w, f32 clip_a).  Version 1 (default) is the reference's
  layout byte for byte (Dense weights are [out, in] like layers.cpp:132), so
  either side loads the other's files.  What exact resume needs and v1
  lacks -- the LCG gradient-stream state, the iteration counter and the
  momentum buffers -- goes to a sidecar file "<path>.resume" (or, with
  version=2, after the clip records of the same file; the reference rejects
  version 2).
* Trace CSV (csv.cpp:8-27): header row, one row per iteration
  per quantised layer: run_id, iter, layer, loss, dc, clip, lr_scale,
  eps_norm, ghat_sqnorm; floats with 9 significant digits, LF endings.
"""
from __future__ import annotations

import struct

import torch

from ._lib import DsgcView

MAGIC = b"I8FT"


def _tensors(trainer):
    out = {}
    for path, layer in trainer.leaves:
        for p in layer.params():
            out[f"{path}.{p.name}"] = p.value
        for b in layer.buffers():
            out[f"{path}.{b.name}"] = b.value
    return dict(sorted(out.items(), key=lambda kv: kv[0].encode()))


RESUME_MAGIC = b"I8RS"


def _resume_blob(trainer, iteration):
    mom = trainer.mflat
    head = struct.pack("<Iq", int(trainer.grad_stream.item()) & 0xFFFFFFFF, iteration)
    body = struct.pack("<q", 0 if mom is None else mom.numel())
    if mom is not None:
        body += mom.cpu().numpy().tobytes()
    return head, body


def save_checkpoint(trainer, path: str, iteration: int = 0, version: int = 1, resume: bool = True):
    tensors = _tensors(trainer)
    views = trainer.arena.read_views()
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<III", version, len(tensors), len(trainer.quant_layers)))
        for name, t in tensors.items():
            nb = name.encode()
            f.write(struct.pack("<I", len(nb)) + nb)
            f.write(struct.pack("<I", t.dim()) + struct.pack(f"<{t.dim()}I", *t.shape))
            f.write(t.detach().float().contiguous().cpu().numpy().tobytes())
        for (lpath, layer), v in zip(trainer.quant_layers, views):
            nb = lpath.encode()
            qs = layer.qs
            f.write(struct.pack("<I", len(nb)) + nb)
            f.write(struct.pack("<fdqqff", v.clip, v.last_dc, v.iter_of_last_update, v.period,
                                float(qs.clip_w.item()), float(qs.clip_a.item())))
        head, body = _resume_blob(trainer, iteration)
        if version >= 2:
            f.write(head)
    if version == 1 and resume:
        with open(path + ".resume", "wb") as r:
            r.write(RESUME_MAGIC + head + body)


def load_checkpoint(trainer, path: str) -> int:
    """Restores parameters, buffers, clip states (and for v2, or a v1 file
    with its .resume sidecar, the LCG state and momentum); returns the saved
    iteration (0 for a bare v1 file, e.g. one the reference wrote)."""
    tensors = _tensors(trainer)
    by_layer = {p: l for p, l in trainer.quant_layers}
    idx = {p: i for i, (p, _) in enumerate(trainer.quant_layers)}
    views = trainer.arena.read_views()
    with open(path, "rb") as f:
        if f.read(4) != MAGIC:
            raise RuntimeError("checkpoint: bad magic")
        version, n_t, n_c = struct.unpack("<III", f.read(12))
        if version not in (1, 2):
            raise RuntimeError("checkpoint: unsupported version")
        for _ in range(n_t):
            (ln,) = struct.unpack("<I", f.read(4))
            name = f.read(ln).decode()
            (rank,) = struct.unpack("<I", f.read(4))
            dims = struct.unpack(f"<{rank}I", f.read(4 * rank))
            if name not in tensors:
                raise RuntimeError(f"checkpoint: unknown tensor {name}")
            t = tensors[name]
            if tuple(dims) != tuple(t.shape):
                raise RuntimeError(f"checkpoint: shape mismatch for {name}")
            buf = f.read(4 * t.numel())
            t.copy_(torch.frombuffer(bytearray(buf), dtype=torch.float32).view(t.shape))
        for _ in range(n_c):
            (ln,) = struct.unpack("<I", f.read(4))
            name = f.read(ln).decode()
            if name not in by_layer:
                raise RuntimeError(f"checkpoint: unknown clip state {name}")
            clip, last_dc, itl, period, cw, ca = struct.unpack("<fdqqff", f.read(4 + 8 + 8 + 8 + 4 + 4))
            layer = by_layer[name]
            v = views[idx[name]]
            v.clip, v.last_dc, v.iter_of_last_update, v.period = clip, last_dc, itl, period
            layer.qs.dsgc.write(v)
            layer.qs.clip_w.fill_(cw)
            layer.qs.clip_a.fill_(ca)
            layer.qs.clip_w_set = cw > 0
            layer.qs.clip_a_set = ca > 0
        it = 0
        if version >= 2:
            state, it = struct.unpack("<Iq", f.read(12))
            trainer.grad_stream.fill_(struct.unpack("<i", struct.pack("<I", state))[0])
    side = path + ".resume"
    import os
    if version == 1 and os.path.exists(side):
        with open(side, "rb") as r:
            if r.read(4) != RESUME_MAGIC:
                raise RuntimeError("checkpoint: bad resume sidecar")
            state, it = struct.unpack("<Iq", r.read(12))
            trainer.grad_stream.fill_(struct.unpack("<i", struct.pack("<I", state))[0])
            (nm,) = struct.unpack("<q", r.read(8))
            if nm:
                if trainer.mflat is None or trainer.mflat.numel() != nm:
                    raise RuntimeError("checkpoint: momentum buffer does not match the trainer")
                trainer.mflat.copy_(torch.frombuffer(bytearray(r.read(4 * nm)), dtype=torch.float32))
    return it


def fmt_sig9(v: float) -> str:
    return "%.9g" % v


class CsvTrace:
    """TraceSink writing the reference's trace CSV."""
    HEADER = ["run_id", "iter", "layer", "loss", "dc", "clip", "lr_scale", "eps_norm", "ghat_sqnorm"]

    def __init__(self, path: str):
        self.f = open(path, "w", newline="\n")
        self.f.write(",".join(self.HEADER) + "\n")

    def row(self, run_id, it, layer, loss, dc, clip, lr_scale, eps_norm, ghat_sqnorm):
        cells = [run_id, str(it), layer] + [fmt_sig9(x) for x in (loss, dc, clip, lr_scale, eps_norm, ghat_sqnorm)]
        self.f.write(",".join(cells) + "\n")

    def report(self, run_id, rep):
        for ls in rep.layers:
            self.row(run_id, rep.iter, ls.layer, rep.loss, ls.dc, ls.clip, ls.lr_scale, ls.eps_norm, ls.ghat_sqnorm)

    def close(self):
        self.f.close()
