"""GPU: the data-parallel device path with two ranks sharing
cuda:0 over gloo.  Each rank runs the real gradient quantiser (K3 + the DSGC
search on iteration 0, the measurement pass on iteration 1) on its contiguous
batch shard with the allreduce hook and the shard offset installed
(i8t_ctx_set_allreduce / i8t_ctx_set_shard).  The concatenated int8 payloads,
the clip, d_c and the LCG stream must equal one device quantising the whole
batch -- bit-exact; and the int64 wgrad accumulators summed over the ranks
must equal the whole-batch accumulator."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grad(n, c, h, seed):
    rng = np.random.default_rng(seed)
    g = rng.laplace(0.0, 1e-4, (n, h, h, c)).astype(np.float32)
    g[rng.random(g.shape) < 0.01] *= 40.0
    g[rng.random(g.shape) < 0.2] = 0.0
    return g


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C

        from paper_1912_12607_b200 import ops
        from paper_1912_12607_b200.trainer import _DistHook
        torch.cuda.set_device(0)
        hook = _DistHook()
        ops.call("i8t_ctx_set_allreduce", ops.ctx(), C.cast(hook.cfn, C.c_void_p), None)
        ops.call("i8t_ctx_set_shard", ops.ctx(), rank, world)
        N, Cc, H = 8, 64, 14
        g = _grad(N, Cc, H, 7)
        b = N // world
        gl = torch.from_numpy(np.ascontiguousarray(g[rank * b:(rank + 1) * b])).cuda()
        st = ops.DsgcState(period=100)
        lcg = ops.new_lcg_state(12345)
        qs = []
        for it in range(2):
            qs.append(ops.quantize_gradient(st, gl, it, lcg, nhwc=True).cpu().numpy())
        v = st.view()
        # wgrad accumulator of this shard: 1x1 conv, activations of the shard
        rng = np.random.default_rng(3)
        a = rng.integers(-127, 128, (N, H, H, 64)).astype(np.int8)[rank * b:(rank + 1) * b]
        geo = ops.geom(b, 64, H, H, Cc, 1, 1, 1, 0)
        qg = torch.from_numpy(qs[1]).cuda()
        acc = torch.empty((64, Cc), dtype=torch.int64, device="cuda")
        one = torch.ones(1, device="cuda")
        ops.conv_wgrad_nhwc(geo, qg, Cc, torch.from_numpy(a).cuda(), 64, one, one, acc=acc)
        dist.all_reduce(acc, op=dist.ReduceOp.SUM)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), q0=qs[0], q1=qs[1], clip=v.clip, dc=v.last_dc,
                 eps=v.eps_norm, lcg=ops.lcg_value(lcg), acc=acc.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_data_parallel_quantiser_equals_single_device(ops, tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ranks = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    # single device, whole batch (hooks off in this process)
    N, Cc, H = 8, 64, 14
    g = torch.from_numpy(_grad(N, Cc, H, 7)).cuda()
    st = ops.DsgcState(period=100)
    lcg = ops.new_lcg_state(12345)
    q0 = ops.quantize_gradient(st, g, 0, lcg, nhwc=True).cpu().numpy()
    q1 = ops.quantize_gradient(st, g, 1, lcg, nhwc=True).cpu().numpy()
    v = st.view()
    np.testing.assert_array_equal(np.concatenate([r["q0"] for r in ranks]), q0)
    np.testing.assert_array_equal(np.concatenate([r["q1"] for r in ranks]), q1)
    for r in ranks:
        assert float(r["clip"]) == v.clip
        assert int(r["lcg"]) == ops.lcg_value(lcg)
        np.testing.assert_allclose(float(r["dc"]), v.last_dc, rtol=0, atol=1e-12)
        np.testing.assert_allclose(float(r["eps"]), v.eps_norm, rtol=1e-12)
    rng = np.random.default_rng(3)
    a = rng.integers(-127, 128, (N, H, H, 64)).astype(np.int8)
    acc = torch.empty((64, Cc), dtype=torch.int64, device="cuda")
    one = torch.ones(1, device="cuda")
    ops.conv_wgrad_nhwc(ops.geom(N, 64, H, H, Cc, 1, 1, 1, 0), torch.from_numpy(q1).cuda(), Cc,
                        torch.from_numpy(a).cuda(), 64, one, one, acc=acc)
    for r in ranks:
        np.testing.assert_array_equal(r["acc"], acc.cpu().numpy())


def test_nccl_communicator_in_the_context(ops):
    """The library-owned NCCL communicator (comm.cu) on a world of one: the
    statistics go through ncclAllGather + the fixed-order fold on the stream;
    quantiser results must equal the communicator-free path bit for bit."""
    import ctypes as C
    g = torch.from_numpy(_grad(4, 64, 14, 9)).cuda()

    def run():
        st = ops.DsgcState(period=100)
        lcg = ops.new_lcg_state(5)
        q = [ops.quantize_gradient(st, g, it, lcg, nhwc=True).cpu().numpy() for it in range(2)]
        v = st.view()
        return q, (v.clip, v.last_dc, v.eps_norm, v.ghat_sqnorm), ops.lcg_value(lcg)
    n0 = ops.launch_count()
    ref = run()
    n_ref = ops.launch_count() - n0
    raw = (C.c_uint8 * 128)()
    ops.call("i8t_nccl_unique_id", C.cast(raw, C.c_void_p), 128)
    ops.call("i8t_ctx_set_nccl", ops.ctx(), C.cast(raw, C.c_void_p), 128, 0, 1)
    try:
        n0 = ops.launch_count()
        got = run()
        n_comm = ops.launch_count() - n0
    finally:
        ops.call("i8t_ctx_set_nccl", ops.ctx(), None, 0, 0, 1)
    assert n_comm > n_ref  # the statistics really went through the communicator (one fold per phase)
    for a, b in zip(ref[0], got[0]):
        np.testing.assert_array_equal(a, b)
    assert ref[1:] == got[1:]
