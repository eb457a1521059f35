"""Launch one conv direction on one shape a few times (for ncu captures).
    python tools/conv_one.py --mode fwd --shape 256,64,56,256,1,1,0 --reps 3
shape = n,c,h,k,kernel,stride,pad"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12607_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="fwd", choices=["fwd", "dgrad", "wgrad"])
ap.add_argument("--shape", default="256,64,56,256,1,1,0")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
n, c, h, k, kk, s, p = (int(v) for v in a.shape.split(","))
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
for _ in range(a.reps):
    if a.mode == "fwd":
        ops.conv_fwd_nhwc(g, qa, cp, qw, qw.shape[1], one, one, z_out=z)

    elif a.mode == "dgrad":
        ops.conv_dgrad_nhwc(g, qg, kp, qwt, qwt.shape[1], one, one, out=ga)
    else:
        ops.conv_wgrad_nhwc(g, qg, kp, qa, cp, one, one, acc=acc, gw=gw)
torch.cuda.synchronize()
print("done")
