"""Run the ResNet 3x3 64->64 @56 batch-32 sparse conv (conv-ordered weights,
rotating input sets like scripts/sweep.py) for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
C, H, Kf, R, pad, Nb, V = 64, 56, 64, 3, 1, 32, 64
crs = C * R * R
mask = torch.from_numpy(bench.synth_mask(Kf, crs, V, crs // 4, 1234)).to(dev)
n = 12
geo = sb.ConvGeometry(R, R, 1, pad)
ws = [sb.conv_prepare(sb.compress_shflbw(bench.uniform16(torch, (Kf, crs), 100 + s, dev), mask, V), geo)
      for s in range(n)]
xs = [bench.uniform16(torch, (C, H, H, Nb), 300 + s, dev) for s in range(n)]
outs = [torch.empty((Kf, H, H, Nb), dtype=torch.bfloat16, device=dev) for _ in range(n)]
lib = sb.shflbw._lib()
for it in range(3 * n):
    k = it % n
    assert lib.shflbw_cu_conv2d(ws[k].ptr, xs[k].data_ptr(), C, H, H, Nb, R, R, 1, pad, outs[k].data_ptr(), 1,
                                torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
print("conv profile run ok")
