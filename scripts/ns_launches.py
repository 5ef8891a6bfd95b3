"""Development: a short chain of north-star SpMMs on rotating operand sets
(for an ncu capture of one launch)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402

wl = dict(bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "ns"])
M, N, K, V, alpha = wl["M"], wl["N"], wl["K"], wl["V"], wl["alpha"]
dev = torch.device("cuda", 0)
mask = torch.from_numpy(bench.synth_mask(M, K, V, int(round(alpha * K)), 1234)).to(dev)
mats = [sb.compress_shflbw(bench.uniform16(torch, (M, K), 100 + i, dev), mask, V) for i in range(4)]
Bs = [bench.uniform16(torch, (K, N), 200 + i, dev) for i in range(4)]
Cs = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(4)]
for i in range(24):
    sb.spmm_execute(mats[i % 4], Bs[i % 4], out=Cs[i % 4])
torch.cuda.synchronize()
print(sb.last_plan())
