"""Time the tcgen05 conv kernel on GEMM-shaped 1x1 problems (CUDA events,
median of 20) to compare its mainloop with a library GEMM at the same size
(tools/cutlass_int8_ref.py).  usage: python tools/conv_gemm_probe.py [M C K]..."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_12607_b200 import ops  # noqa: E402

shapes = [tuple(int(v) for v in s.split(",")) for s in sys.argv[1:]] or [(8192, 8192, 8192), (8192, 8192, 256),
                                                                         (32768, 2048, 512), (50176, 2304, 256)]
for m, c, k in shapes:
    g = ops.geom(1, c, 1, m, k, 1, 1, 1, 0)  # 1x1 conv over m pixels = GEMM [m x c] . [c x k]
    qa = torch.randint(-127, 128, (m, c), dtype=torch.int8, device="cuda")
    w = torch.randn(k, c, 1, 1, device="cuda")
    qw, _ = ops.quantize_weight(w, float(w.abs().max()), c_pad=c, k_pad=k)
    one = torch.ones(1, device="cuda")
    z = torch.empty((m, k), device="cuda")
    ts = []
    for i in range(6):  # 20 back-to-back launches queued behind a GPU sleep: no host gaps inside the events
        torch.cuda._sleep(20_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            ops.conv_fwd_nhwc(g, qa, c, qw, qw.shape[1], one, one, z_out=z)
        e1.record()
        e1.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1) / 20)
    t = statistics.median(ts)
    print(f"M={m} C={c} K={k}: {t * 1e3:.1f} us  {2 * m * c * k / t / 1e9:.0f} TOPS  "
          f"(fp32 out {m * k * 4 / t / 1e6:.0f} GB/s)", flush=True)
