"""Microbenchmark of the BN column reductions (i8t_bn_fwd_stats = k_bn_colsum<0>,
i8t_bn_bwd_reduce = k_bn_colsum<1>) on ResNet-50 activation shapes (batch 256)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12607_b200 import ops  # noqa: E402


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for m, c in [(256 * 112 * 112, 64), (256 * 3136, 64), (256 * 3136, 256), (256 * 784, 128), (256 * 784, 512),
             (256 * 196, 256), (256 * 196, 1024), (256 * 49, 512), (256 * 49, 2048)]:
    z = torch.randn(m, c, device="cuda")
    g = torch.randn(m, c, device="cuda") * 1e-3
    gamma, beta = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")
    bn = torch.zeros(6 * c, dtype=torch.float64, device="cuda")
    gg, gb = torch.zeros(c, device="cuda"), torch.zeros(c, device="cuda")
    f0 = lambda: ops.call("i8t_bn_fwd_stats", ops.ctx(), ops._p(z), m, c, C.c_double(0.1), C.c_double(1e-5),
                          ops._p(bn), None, None)
    f1 = lambda: ops.call("i8t_bn_bwd_reduce", ops.ctx(), ops._p(g), ops._p(z), m, c, ops._p(bn), ops._p(gamma),
                          ops._p(beta), 1, None, ops._p(gg), ops._p(gb))
    t0, t1 = timeit(f0), timeit(f1)
    print(f"m={m:9d} c={c:5d}  fwd_stats {t0 * 1e3:8.1f} us {4 * m * c / t0 / 1e6:7.0f} GB/s   "
          f"bwd_reduce {t1 * 1e3:8.1f} us {8 * m * c / t1 / 1e6:7.0f} GB/s", flush=True)
