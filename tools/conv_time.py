"""Time one conv direction on one shape (CUDA events, L2 flushed between reps).
    python tools/conv_time.py fwd 256,256,14,256,3,1,1 [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12607_b200 import ops  # noqa: E402

mode, shape = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
n, c, h, k, kk, s, p = (int(v) for v in shape.split(","))
g = ops.geom(n, c, h, h, k, kk, kk, s, p)
P, Q = g.out_hw()
cp, kp = ops.pad4(c), ops.pad4(k)
qa = torch.randint(-127, 128, (n, h, h, cp), dtype=torch.int8, device="cuda")
qg = torch.randint(-127, 128, (n, P, Q, kp), dtype=torch.int8, device="cuda")
w = torch.randn(k, c, kk, kk, device="cuda")
qw, qwt = ops.quantize_weight(w, float(w.abs().max()), c_pad=cp, k_pad=kp)
one = torch.ones(1, device="cuda")
z = torch.empty((n * P * Q, k), device="cuda")
ga = torch.empty((n * h * h, c), device="cuda")
acc = torch.empty((kk * kk * cp, k), dtype=torch.int64, device="cuda")
gw = torch.empty((k, c, kk, kk), device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")


def run():
    if mode == "fwd":
        ops.conv_fwd_nhwc(g, qa, cp, qw, qw.shape[1], one, one, z_out=z)
    elif mode == "dgrad":
        ops.conv_dgrad_nhwc(g, qg, kp, qwt, qwt.shape[1], one, one, out=ga)
    else:
        ops.conv_wgrad_nhwc(g, qg, kp, qa, cp, one, one, acc=acc, gw=gw)


for _ in range(3):
    run()
ts = []
for _ in range(reps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"{mode} {shape} env BN={os.environ.get('I8T_FORCE_BN', '-')}: {ts[len(ts) // 2]:.1f} us")
