"""Stem max pool (BN + ReLU fused) at ResNet-50 b256: 256 x 112 x 112 x 64 fp32
-> 56 x 56, CUDA events per launch.  I8T_NO_POOL_RUN=1 selects the per-window
kernel."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12607_b200 import ops  # noqa: E402

n, h, w, c = 256, 112, 112, 64
x = torch.randn(n * h * w, c, device="cuda")
bn = torch.zeros(6 * c, dtype=torch.float64, device="cuda")
bn[c:2 * c] = 1.0
gamma, beta = torch.ones(c, device="cuda"), torch.zeros(c, device="cuda")
y = torch.empty((n, 56, 56, c), device="cuda")
idx = torch.empty((n, 56, 56, c), dtype=torch.uint8, device="cuda")
f = lambda: ops.call("i8t_maxpool_fwd", ops.ctx(), ops._p(x), n, h, w, c, 3, 2, 1, ops._p(bn), ops._p(gamma),
                     ops._p(beta), 1, ops._p(y), ops._p(idx))
for _ in range(3):
    f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    f()
e.record()
torch.cuda.synchronize()
t = s.elapsed_time(e) / 10 * 1e3
b = x.numel() * 4 + y.numel() * 5
print(f"maxpool_fwd {t:.1f} us  {b / t / 1e3:.0f} GB/s")
