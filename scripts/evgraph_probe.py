import torch
x = torch.randn(1 << 20, device="cuda")
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True)
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    for _ in range(3): x.mul_(1.0001)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    for _ in range(10): x.mul_(1.0001)
    e0.record(s)
    for _ in range(20): x.mul_(1.0001)
    e1.record(s)
for _ in range(3):
    g.replay(); torch.cuda.synchronize(); print("in-graph events ms", e0.elapsed_time(e1))
