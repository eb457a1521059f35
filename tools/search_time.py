"""Time ops.search_clip (grid R, 2 golden rounds) on a ResNet-50-sized gradient
(205M elements, the largest layer): python tools/search_time.py [R ...].
I8T_DSGC_HIST=0 times the per-candidate grid passes instead of the histogram."""
import sys

import torch

sys.path.insert(0, ".")
from oracle import lib as O  # noqa: E402  (synthetic input only)
from paper_1912_12607_b200 import ops  # noqa: E402

g = torch.from_numpy(O.gradient_like((205_520_896,), 1, 1e-3, 0.01)).cuda()
for R in [int(a) for a in sys.argv[1:]] or [32]:
    ops.search_clip(g, R, 2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        r = ops.search_clip(g, R, 2)
    e1.record()
    torch.cuda.synchronize()
    print(f"R {R} search_clip {e0.elapsed_time(e1) / 5:.3f} ms -> {r}")
