"""Per-launch cost of a chain of tiny dependent kernels on one stream, eager vs
CUDA-graph replay (the floor a ~500-launch training step pays per launch)."""
import torch, time
x = torch.zeros(1024, device="cuda")
def chain(n):
    for _ in range(n):
        x.add_(1.0)
for _ in range(3): chain(500)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); chain(500); e.record(); torch.cuda.synchronize()
print("eager tiny kernel: %.2f us/launch" % (s.elapsed_time(e) * 1e3 / 500))
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    chain(10)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    chain(500)
g.replay(); torch.cuda.synchronize()
s.record(); g.replay(); e.record(); torch.cuda.synchronize()
print("graph tiny kernel: %.2f us/launch" % (s.elapsed_time(e) * 1e3 / 500))
