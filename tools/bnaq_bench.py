"""i8t_bn_act_quant (BN apply + ReLU + the next conv's nearest quantiser) on
ResNet-50 inner-BN shapes (batch 256): time per launch (CUDA events)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12607_b200 import ops  # noqa: E402

for m, c in [(256 * 3136, 64), (256 * 784, 128), (256 * 196, 256), (256 * 49, 512), (256 * 3136, 128)]:
    z = torch.randn(m, c, device="cuda")
    gamma, beta = torch.rand(c, device="cuda") + 0.5, torch.randn(c, device="cuda") * 0.1
    bn = torch.zeros(6 * c, dtype=torch.float64, device="cuda")
    ops.call("i8t_bn_fwd_stats", ops.ctx(), ops._p(z), m, c, C.c_double(0.1), C.c_double(1e-5), ops._p(bn), None, None)
    clip = torch.tensor([3.0], device="cuda")
    q = torch.empty((m, c), dtype=torch.int8, device="cuda")
    f = lambda: ops.call("i8t_bn_act_quant", ops.ctx(), ops._p(z), m, c, ops._p(bn), ops._p(gamma), ops._p(beta), 1,
                         ops._p(clip), ops._p(q), None)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        f()
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / 20 * 1e3
    print(f"m={m:8d} c={c:4d} {t:7.1f} us  {5 * m * c / t / 1e3:6.0f} GB/s", flush=True)
