"""World-size-2 gloo tests of the data-parallel host logic (CPU).

Each rank quantises its batch shard with the oracle standing in for the
device kernel (test-only), drawing from the global stream at
dp.shard_draw_offset and using global statistics from dp.combine_totals;
the gathered result must equal the single-device quantisation of the whole
batch bit-for-bit, the stream must advance by dp.layer_draws, and the int64
weight-gradient allreduce must equal the whole-batch wgrad accumulator."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import lib as O
        from paper_1912_12607_b200 import dp

        N, C, H = 8, 8, 6
        g = O.gradient_like((N, C, H, H), 5, 1e-3, 0.02)
        gl = dp.shard_batch(torch.from_numpy(g), rank, world).numpy()
        # global statistics: max|g| (MAX) + sum g^2 (SUM) as the device totals buffer would carry them
        tot = torch.tensor([float(np.abs(gl).max()), float((gl.astype(np.float64) ** 2).sum())], dtype=torch.float64)
        tot2 = tot.clone()
        dp.combine_totals(tot)
        dp.combine_totals_gather(tot2)  # the one-collective form the device hook uses (op 2)
        assert float(tot2[0]) == float(tot[0])
        assert abs(float(tot2[1]) - float(tot[1])) <= 1e-12 * abs(float(tot[1]))
        clip = float(np.float32(tot[0].item()) * np.float32(0.5))
        # stochastic draws from the global stream at this shard's offset
        seed = 1234
        start = O.lcg_jump(seed, dp.shard_draw_offset(rank, gl.size))
        q_local, _ = O.quantize(gl, clip, True, start)
        after = O.lcg_jump(seed, dp.layer_draws(world, gl.size))
        # wgrad as int64, summed across ranks
        qa = np.random.default_rng(7).integers(-127, 128, (N, C, H, H)).astype(np.int8)
        qal = dp.shard_batch(torch.from_numpy(qa), rank, world).numpy()
        geo = O.geom(N // world, C, H, H, C, 3, 3, 1, 1)
        acc, _ = O.conv_wgrad(q_local, qal, geo, O.quant_scale(clip), 1.0)
        acc_t = torch.from_numpy(acc.copy())
        dp.allreduce_int64_(acc_t)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), q=q_local, tot=tot.numpy(), clip=clip, after=after,
                 acc=acc_t.numpy())
    finally:
        dist.destroy_process_group()


def test_dp_two_ranks_match_single_device(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    from oracle import lib as O
    r = [np.load(tmp_path / f"r{i}.npz") for i in range(world)]
    N, C, H = 8, 8, 6
    g = O.gradient_like((N, C, H, H), 5, 1e-3, 0.02)
    # global statistics identical on every rank and equal to the whole-batch values
    for x in r:
        assert x["tot"][0] == np.float32(np.abs(g).max())
        assert x["tot"][1] == pytest.approx(float((g.astype(np.float64) ** 2).sum()), rel=1e-12)
    clip = float(r[0]["clip"])
    q_full, stream_after = O.quantize(g, clip, True, 1234)
    np.testing.assert_array_equal(np.concatenate([x["q"] for x in r]), q_full)
    assert all(int(x["after"]) == stream_after for x in r)
    qa = np.random.default_rng(7).integers(-127, 128, (N, C, H, H)).astype(np.int8)
    acc_full, _ = O.conv_wgrad(q_full, qa, O.geom(N, C, H, H, C, 3, 3, 1, 1), O.quant_scale(clip), 1.0)
    for x in r:
        np.testing.assert_array_equal(x["acc"], acc_full)


def test_shard_offsets_wrap_mod_2_32():
    from paper_1912_12607_b200 import dp
    assert dp.shard_draw_offset(3, 2 ** 31) == (3 * 2 ** 31) % 2 ** 32
    assert dp.layer_draws(8, 2 ** 30) == 0
    with pytest.raises(ValueError):
        dp.shard_batch(torch.zeros(5, 2), 0, 2)
