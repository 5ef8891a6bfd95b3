"""Development: one north-star and one large-FFN asynchronous conversion
(for an ncu launch list of the converter's kernels)."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402
dev = torch.device("cuda", 0)
for M, K, V in ((2048, 2048, 64), (16384, 4096, 64)):
    mask = torch.from_numpy(bench.synth_mask(M, K, V, K // 4, 1234)).to(dev)
    W = bench.uniform16(torch, (M, K), 100, dev)
    a, st = sb.compress_shflbw_async(W, mask, V)
    torch.cuda.synchronize()
    sb.compress_shflbw_async(W, mask, V, out=a, status=st)
    torch.cuda.synchronize()
    sb.finalize(a, st)
print("ok")
