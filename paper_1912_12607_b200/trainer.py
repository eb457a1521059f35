"""Per-step INT8 trainer on the device -- Trainer (train.hpp:66-92,
train.cpp:12-120): cosine base LR, INT8 forward with activation-amax
tracking, softmax-CE in double, divergence check, backward in the reference's
layer order drawing from one device-resident LCG gradient stream, bad-gradient
check, SGD with the per-layer DCLR factor phi(d_c), periodic refresh of the
weight / activation clips.

Data parallel: one process per GPU, batch sharded; the DSGC
statistics are all-reduced through the C-ABI hook so every rank quantises the
global gradient exactly as one device would; the int64 weight-gradient
accumulators are all-reduced (exact) before the FP64 rescale; FP32 parameter
gradients (BN, fc bias) are averaged-free summed like the reference's single
batch sum.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import dp, ops
from ._lib import DsgcView, WqDesc, call
from .layers import (BackwardCtx, Conv2d, Dense, ForwardCtx, Mode, SoftmaxCrossEntropy, StateArena, int8_replace,
                     leaves)


@dataclass
class TrainConfig:
    """TrainConfig (train.hpp:17-32)."""
    mode: Mode = Mode.INT8
    base_lr: float = 0.1
    schedule: str = "cosine"
    alpha: float = 20.0
    beta: float = 0.1
    form: str = "exp"
    lr_scaling_enabled: bool = True
    grid_resolution: int = 32
    refine_rounds: int = 2
    clip_enabled: bool = True
    clip_period: int = 100
    seed: int = 1
    batch_size: int = 64
    epochs: int = 5
    calibration_batches: int = 2
    momentum: float = 0.0  # SGD momentum (train.cpp:106-111), one flat device buffer per trainer


@dataclass
class LayerStepStat:
    layer: str
    dc: float = 0.0
    clip: float = 0.0
    lr_scale: float = 1.0
    eps_norm: float = 0.0
    ghat_sqnorm: float = 0.0


@dataclass
class StepReport:
    iter: int = 0
    loss: float = 0.0
    diverged: bool = False
    base_lr_t: float = 0.0
    layers: list = field(default_factory=list)


class _DistHook:
    """i8t_allreduce_fn implemented with torch.distributed on raw device buffers."""

    FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p)

    def __init__(self):
        self.cfn = self.FN(self._call)

    @staticmethod
    def _view_i32(ptr):
        class _A:
            __cuda_array_interface__ = {"shape": (1,), "typestr": "<i4", "data": (int(ptr), False), "version": 3}
        return torch.as_tensor(_A(), device="cuda")

    @staticmethod
    def _view(ptr, count):
        class _A:
            __cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8", "data": (int(ptr), False),
                                        "version": 3}
        return torch.as_tensor(_A(), device="cuda")

    def _call(self, user, buf, count, dtype, op, stream):
        try:
            t = self._view(buf, count)
            if op == 2:  # [0] MAX, [1:] SUM in one collective: gather every rank's row, fold locally
                dp.combine_totals_gather(t)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM)
            return 0
        except Exception:  # pragma: no cover - surfaced as I8T_ECUDA by the library
            return 1


# Weight gradients on a side stream overlapping the backward-data chain
# (single device; I8T_WGRAD_STREAM=0 keeps them in line).
WGRAD_STREAM = os.environ.get("I8T_WGRAD_STREAM", "1") == "1"


class Trainer:
    def __init__(self, model, cfg: TrainConfig, device="cuda", force_dp_hook: bool = False):
        self.model, self.cfg = model, cfg
        self.leaves = leaves(model.net)
        self.quant_layers = [(p, l) for p, l in self.leaves if l.qs is not None]
        self.arena = StateArena(device)
        for path, layer in self.quant_layers:
            layer.qs.layer_id = path
            self.arena.register(layer)
        self.arena.build(cfg.clip_period)
        # Trainer::grad_stream_(uint32(seed)) (train.cpp:13)
        self.grad_stream = ops.new_lcg_state(cfg.seed & 0xFFFFFFFF, device)
        self.world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
        self.rank = dist.get_rank() if self.world > 1 else 0
        self._hook = None
        self._wgrad_side = None  # side stream of the weight gradients (single device)
        self.device = device
        if self.world > 1 or force_dp_hook:  # force: exercise the data-parallel phases at world size 1
            if self.world > 1 and dist.get_backend() == "nccl" and os.environ.get("I8T_DP_COMM", "nccl") == "nccl":
                # the library's own NCCL communicator combines the DSGC statistics
                # on the compute stream (no host callback inside the backward)
                self._hook = "nccl"
                ident = torch.zeros(128, dtype=torch.uint8, device=device)
                if self.rank == 0:
                    raw = (C.c_uint8 * 128)()
                    call("i8t_nccl_unique_id", C.cast(raw, C.c_void_p), 128)
                    ident.copy_(torch.tensor(list(raw), dtype=torch.uint8))
                dist.broadcast(ident, 0)
                raw = (C.c_uint8 * 128)(*ident.cpu().tolist())
                call("i8t_ctx_set_nccl", ops.ctx(), C.cast(raw, C.c_void_p), 128, self.rank, self.world)
            else:  # gloo (tests) or I8T_DP_COMM=python: torch.distributed through a host callback
                self._hook = _DistHook()
                call("i8t_ctx_set_allreduce", ops.ctx(), C.cast(self._hook.cfn, C.c_void_p), None)
                call("i8t_ctx_set_shard", ops.ctx(), self.rank, self.world)
        # the gradient w.r.t. the input images is discarded: the first conv skips backward-data
        first = self.leaves[0][1]
        if hasattr(first, "need_input_grad"):
            first.need_input_grad = False
        self.skip = torch.zeros(1, dtype=torch.int32, device=device)
        # divergence (train.cpp:73-77) is decided on the device: the backward runs
        # regardless and a diverged step restores what it mutated (DSGC states,
        # LCG stream, latched error word) from a pre-backward snapshot -- no host
        # sync inside the step
        self.div = torch.zeros(1, dtype=torch.int32, device=device)
        self._snap_arena = torch.empty_like(self.arena.buf)
        self._snap_lcg = torch.empty_like(self.grad_stream)
        self._snap_err = torch.empty(4, dtype=torch.int32, device=device)
        ptr = C.POINTER(C.c_int32)()
        call("i8t_ctx_error_word", ops.ctx(), C.byref(ptr))
        self._err = _DistHook._view_i32(C.cast(ptr, C.c_void_p).value)
        self._wq_buf, self._wq_n = None, 0  # device i8t_wq_desc array (built at the second step)
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=device)
        self.graph_replayed_launches = 0
        self.lr_dev = torch.zeros(1, dtype=torch.float64, device=device)
        self._build_param_arenas(device)
        if self.world > 1:  # identical initial parameters on every rank (seeded alike; made certain)
            dist.broadcast(self.pflat, 0)

    def _build_param_arenas(self, device):
        """Every parameter / gradient becomes a view into one flat arena
        (segments padded to 4 floats) so the bad-gradient scan and the DCLR
        SGD step are one launch each."""
        cfg = self.cfg
        segs, total = [], 0
        # quantised layers' parameters first: their gradients are reduced as
        # integer sums (int64 wgrad accumulators, the fc bias's int8 column
        # sums), the rest (FP32 BN gradients) form one tail slice that a
        # data-parallel step all-reduces in a single collective
        attrs = [(layer, owner, va, ga) for _, layer in self.leaves for owner, va, ga in layer.param_attrs()]
        exact = lambda t: t[0].quantized and (t[2] == "weight" or isinstance(t[0], Dense))  # noqa: E731
        q = [t for t in attrs if exact(t)]  # int64-reduced under DP: conv / fc weights, fc bias (integer sums)
        rest = [t for t in attrs if not exact(t)]
        for layer, owner, va, ga in q + rest:
            v = getattr(owner, va)
            segs.append((layer, owner, va, ga, total, v.numel(), v.shape))
            total += (v.numel() + 3) // 4 * 4
            if (layer, owner, va, ga) == (q[-1] if q else None):
                self.fp32_grad_off = total
        if not q or cfg.mode != Mode.INT8:  # FP32 mode: every gradient is an FP32 sum
            self.fp32_grad_off = 0
        self.pflat = torch.zeros(total, dtype=torch.float32, device=device)
        self.gflat = torch.zeros(total, dtype=torch.float32, device=device)
        offs, states = [], []
        cfg = self.cfg
        for layer, owner, va, ga, off, n, shape in segs:
            self.pflat[off: off + n].copy_(getattr(owner, va).reshape(-1))
            setattr(owner, va, self.pflat[off: off + n].view(shape))
            setattr(owner, ga, self.gflat[off: off + n].view(shape))
            offs.append(off)
            use_phi = layer.qs is not None and cfg.mode == Mode.INT8 and layer.quantized and cfg.lr_scaling_enabled
            states.append(layer.qs.dsgc.buf.data_ptr() if use_phi else 0)
        offs.append(total)
        self.seg_off = torch.tensor(offs, dtype=torch.int64, device=device)
        self.seg_state = torch.tensor(states, dtype=torch.int64, device=device)
        self.nseg = len(segs)
        # Trainer::momentum_ (train.cpp:22-26): zero-initialised, one buffer per parameter
        self.mflat = torch.zeros(total, dtype=torch.float32, device=device) if cfg.momentum != 0.0 else None

    # ---------------------------------------------------------------- clips
    def calibrate(self, images):
        """FP32 forward tracking activation maxima (train.cpp:29-32)."""
        self.model.net.forward(images, ForwardCtx(Mode.FP32, training=False, track_amax=True))

    def finish_calibration(self):
        self.refresh_wa_clips()

    def refresh_wa_clips(self):
        """clip_w = max_abs(W) if > 0, clip_a = running max of batch maxima if >
        0, pending_amax reset (train.cpp:36-46), on the device.  A clip left at
        0 (all-zero weights, no calibration batch) keeps its flag clear so the
        forward's lazy max(max_abs, 1e-12) initialisation (layers.cpp:106-107)
        still runs.  One host read for all layers decides the flags."""
        h = ops.ctx()
        for _, layer in self.quant_layers:
            qs = layer.qs
            w = layer.params()[0].value
            call("i8t_max_abs", h, ops._p(w), w.numel(), ops._p(qs.tmp))
            if self.world > 1:
                dist.all_reduce(qs.pending_amax, op=dist.ReduceOp.MAX)
            qs.clip_w.copy_(torch.where(qs.tmp > 0, qs.tmp, qs.clip_w))
            qs.clip_a.copy_(torch.where(qs.pending_amax > 0, qs.pending_amax, qs.clip_a))
            qs.pending_amax.zero_()
        if self.quant_layers:
            clips = torch.stack([torch.cat([l.qs.clip_w, l.qs.clip_a]) for _, l in self.quant_layers]).cpu()
            for (_, layer), (cw, ca) in zip(self.quant_layers, clips.tolist()):
                layer.qs.clip_w_set = cw > 0
                layer.qs.clip_a_set = ca > 0

    def base_lr_at(self, it, total):
        """cosine schedule (train.cpp:48-52)."""
        if self.cfg.schedule == "constant" or total <= 0:
            return self.cfg.base_lr
        return self.cfg.base_lr * 0.5 * (1.0 + math.cos(math.pi * it / total))

    # ---------------------------------------------------------------- step
    def train_step(self, images, labels, it: int, total_iters: int, read_stats: bool = True,
                   _lr_preset: bool = False) -> StepReport:
        """Trainer::train_step (train.cpp:54-120).  images: NHWC float32 CUDA tensor."""
        cfg = self.cfg
        rep = StepReport(iter=it, base_lr_t=self.base_lr_at(it, total_iters))
        wq = cfg.mode == Mode.INT8 and self._quantize_weights_at_once()
        logits = self.model.net.forward(images, ForwardCtx(cfg.mode, True, cfg.mode == Mode.INT8, wq))
        # data parallel: the mean is over the GLOBAL batch (loss summed across ranks when read)
        # the divergence flag (non-finite loss or logits, train.cpp:73-77) comes out of the same pass
        loss, g_logits = SoftmaxCrossEntropy.loss_and_grad(logits, labels, logits.shape[0] * self.world, bad=self.div)
        if self.world > 1:  # every rank takes the same branch
            dist.all_reduce(self.div, op=dist.ReduceOp.MAX)
        self.loss_dev.copy_(loss.reshape(1))
        self._snap_arena.copy_(self.arena.buf)
        self._snap_lcg.copy_(self.grad_stream)
        self._snap_err[:1].copy_(self._err)
        bctx = BackwardCtx(cfg.mode, it, self.grad_stream, cfg.grid_resolution, cfg.refine_rounds, cfg.clip_enabled,
                           cfg.clip_period, cfg.alpha, cfg.beta, cfg.form, cfg.lr_scaling_enabled,
                           self._wgrad_allreduce if self._hook is not None else None)
        if self._hook is None and WGRAD_STREAM and cfg.mode == Mode.INT8:
            if self._wgrad_side is None:
                self._wgrad_side = torch.cuda.Stream(device=self.device)
            bctx.wgrad_stream = self._wgrad_side
        self._wgrad_step_begin()
        self.model.net.backward(g_logits, bctx)
        for work, finalize in bctx.deferred:  # int64 wgrad allreduces issued during the backward
            if work is not None:
                work.wait()
            finalize()
        if bctx.wgrad_stream is not None:  # join the side-stream weight gradients before the update
            torch.cuda.current_stream().wait_stream(bctx.wgrad_stream)
        if self._hook is not None:
            self._wgrad_arena_build()
        if self.world > 1:
            params = [(layer, p) for _, layer in self.leaves for p in layer.params() if p.grad is not None]
            self._allreduce_fp32_grads(params)
        # bad-gradient check (train.cpp:87-95) stays on the device and gates the update,
        # as does the divergence flag
        h = ops.ctx()
        call("i8t_nonfinite_flag", h, ops._p(self.gflat), self.gflat.numel(), ops._p(self.skip))
        self.skip.bitwise_or_(self.div)
        if not _lr_preset:  # a graph replay sets the learning rate of its step before launching
            self.lr_dev.fill_(rep.base_lr_t)
        call("i8t_sgd_dclr_multi", h, ops._p(self.pflat), ops._p(self.gflat), self.nseg, ops._p(self.seg_off),
             ops._p(self.seg_state), C.c_double(rep.base_lr_t), self.lr_dev, ops._p(self.skip), self.mflat,
             C.c_double(cfg.momentum))
        # a diverged step leaves the state as the reference's early return does
        call("i8t_copy_if", h, self.div, self.arena.buf, self._snap_arena, self.arena.buf.numel())
        call("i8t_copy_if", h, self.div, self.grad_stream, self._snap_lcg, 4)
        call("i8t_copy_if", h, self.div, self._err, self._snap_err, 4)
        if read_stats:
            if self.world > 1:
                dist.all_reduce(self.loss_dev, op=dist.ReduceOp.SUM)
            rep.loss = float(self.loss_dev.item())
            rep.diverged = bool(self.skip.item())
            if bool(self.div.item()):  # the host mirrors of the restored DSGC states
                self.sync_states()
            self._read_layer_stats(rep)
        return rep

    # ---------------------------------------------------------------- CUDA graph replay
    def graph_eligible(self, it: int) -> bool:
        """A step can replay the captured graph when it launches exactly what the
        captured step launched: INT8, single device, DSGC search enabled and
        due on no layer (search steps and lazy-clip steps run eagerly), every
        layer's buffers and clips in place (from the third step on)."""
        cfg = self.cfg
        if cfg.mode != Mode.INT8 or not cfg.clip_enabled or self.world > 1 or self._wq_buf is None:
            return False
        return not any(layer.qs.dsgc.due(it) or not (layer.qs.clip_w_set and layer.qs.clip_a_set)
                       for _, layer in self.quant_layers)

    def train_step_graphed(self, images, labels, it: int, total_iters: int, read_stats: bool = False) -> StepReport:
        """train_step replayed from a CUDA graph captured on the first eligible
        step (one graph per input buffer pair), eager otherwise.  The step has
        no host sync, so the ~500 launches of ResNet-50 become one graph launch;
        only the learning rate changes between replays and it is read from
        device memory (lr_dev).  Bit-identical to train_step
        (tests/test_gpu_graph.py)."""
        if not self.graph_eligible(it):
            return self.train_step(images, labels, it, total_iters, read_stats)
        key = (images.data_ptr(), labels.data_ptr())
        graphs = self.__dict__.setdefault("_graphs", {})
        rep = StepReport(iter=it, base_lr_t=self.base_lr_at(it, total_iters))
        self.lr_dev.fill_(rep.base_lr_t)
        if key not in graphs:
            pool = self.__dict__.setdefault("_graph_pool", torch.cuda.graph_pool_handle())
            g = torch.cuda.CUDAGraph()
            n0 = ops.launch_count()
            with torch.cuda.graph(g, pool=pool):
                self.train_step(images, labels, it, total_iters, read_stats=False, _lr_preset=True)
            graphs[key] = (g, ops.launch_count() - n0)
        g, n = graphs[key]
        g.replay()
        self.graph_replayed_launches += n  # this library's kernels inside the replayed graph
        if read_stats:
            rep.loss = float(self.loss_dev.item())
            rep.diverged = bool(self.skip.item())
            if bool(self.div.item()):
                self.sync_states()
            self._read_layer_stats(rep)
        return rep

    def _quantize_weights_at_once(self) -> bool:
        """Every quantised layer's weights in one launch (i8t_quantize_weights_multi)
        once all layers have their buffers and clips (from the second step on)."""
        if self._wq_buf is None:
            convs = [getattr(layer, "conv", layer) for _, layer in self.quant_layers]
            descs = [c.wq_desc() if isinstance(c, Conv2d) else None for c in convs]
            if not descs or any(d is None for d in descs):
                return False
            arr = (WqDesc * len(descs))()
            for a, d in zip(arr, descs):
                ptr = [t.data_ptr() if t is not None else None for t in d[:4]]
                a.w, a.clip, a.q_krsc, a.q_crsk = ptr
                a.k, a.c, a.rs, a.c_pad, a.ld_krsc, a.k_pad, a.ld_crsk, a.src_krsc = d[4:]
            raw = torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8)
            self._wq_buf = raw.to(self.skip.device)
            self._wq_n = len(descs)
        call("i8t_quantize_weights_multi", ops.ctx(), ops._p(self._wq_buf), self._wq_n)
        return True

    def _read_layer_stats(self, rep: StepReport):
        views = self.arena.read_views()
        for (path, layer), v in zip(self.quant_layers, views):
            layer.qs.dsgc.sync(v)
            rep.layers.append(LayerStepStat(path, v.last_dc, v.clip, v.lr_scale, v.eps_norm, v.ghat_sqnorm))

    def sync_states(self):
        """Refresh the host mirrors (clip > 0, iter of last update) from the device."""
        for (_, layer), v in zip(self.quant_layers, self.arena.read_views()):
            layer.qs.dsgc.sync(v)

    # ---------------------------------------------------------------- data parallel
    BUCKET_BYTES = 32 << 20  # int64 wgrad allreduce buckets (launch latency vs overlap)

    def _wgrad_allreduce(self, acc: torch.Tensor):
        """Exact int64 weight-gradient sum across ranks, bucketed.  The first
        data-parallel step reduces layer by layer and records the order in
        which the backward produces the accumulators; from then on every
        layer's accumulator is a view into one int64 arena laid out in that
        order, and a bucket (>= BUCKET_BYTES, or the last layer) is all-reduced
        asynchronously as soon as its last layer is done, overlapping the rest
        of the backward.  The returned handle's wait() covers the layer's bucket."""
        st = self.__dict__.setdefault("_wg", {"order": [], "arena": None})
        if st["arena"] is None:
            st["order"].append(acc)
            return dp.allreduce_int64_(acc, async_op=True)
        i = st["next"]
        st["next"] += 1
        lo, hi = st["slices"][i]
        if acc.data_ptr() != st["arena"][lo:hi].data_ptr():
            raise RuntimeError("data parallel: the backward produced weight gradients in a new order")
        h = st["handles"][i]
        if i == st["bucket_end"][i]:  # last layer of its bucket: launch it
            lo, hi = st["bucket_span"][i]
            h.work = dp.allreduce_int64_(st["arena"][lo:hi], async_op=True)
        return h

    def _wgrad_arena_build(self):
        """After the first data-parallel step: one int64 arena in backward order,
        each layer's accumulator rebound to its slice, buckets fixed."""
        st = self.__dict__.get("_wg")
        if not st or st["arena"] is not None or not st["order"]:
            return
        accs = st["order"]
        owners = {}
        for _, layer in self.quant_layers:
            conv = getattr(layer, "conv", layer)
            if conv.wgrad_acc is not None:
                owners[conv.wgrad_acc.data_ptr()] = conv
        total = sum(a.numel() for a in accs)
        arena = torch.zeros(total, dtype=torch.int64, device=accs[0].device)
        off, spans, ends, b0, bbytes = 0, [], [], 0, 0
        for i, a in enumerate(accs):
            conv = owners[a.data_ptr()]
            conv.wgrad_acc = arena[off: off + a.numel()].view(a.shape)
            off += a.numel()
            bbytes += a.numel() * 8
            if bbytes >= self.BUCKET_BYTES or i == len(accs) - 1:
                for j in range(b0, i + 1):
                    spans.append(None)
                    ends.append(i)
                spans[i] = (sum(x.numel() for x in accs[:b0]), off)
                b0, bbytes = i + 1, 0

        class _Bucket:
            work = None

            def wait(self):
                if self.work is not None:
                    self.work.wait()
        handles = []
        for i in range(len(accs)):
            handles.append(_Bucket() if ends[i] == i else None)
        for i in range(len(accs)):  # layers share their bucket's handle
            handles[i] = handles[ends[i]]
        slices, o = [], 0
        for a in accs:
            slices.append((o, o + a.numel()))
            o += a.numel()
        st.update(arena=arena, bucket_end=ends, bucket_span=spans, handles=handles, slices=slices, next=0)

    def _wgrad_step_begin(self):
        st = self.__dict__.get("_wg")
        if st and st["arena"] is not None:
            st["next"] = 0
            for h in st["handles"]:
                h.work = None

    def _allreduce_fp32_grads(self, params):
        """FP32 parameter gradients (BN gamma / beta, fc bias): one contiguous
        slice of the gradient arena (quantised weights are laid out first)."""
        if self.fp32_grad_off < self.gflat.numel():
            dist.all_reduce(self.gflat[self.fp32_grad_off:], op=dist.ReduceOp.SUM)


def synthetic_batch(model, batch, seed, device="cuda"):
    """Synthetic images N(0,1) NHWC + uniform labels."""
    gen = torch.Generator(device=device).manual_seed(seed)
    c, h, w = model.in_shape
    x = torch.randn((batch, h, w, c), generator=gen, device=device)
    y = torch.randint(0, model.num_classes, (batch,), generator=gen, device=device)
    return x, y
