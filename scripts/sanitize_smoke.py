"""Small invocations of every kernel family for compute-sanitizer runs
(development): converter, 2x2 / persistent / K-split SpMM, conv (both
producers, odd Q), fused multi-destination epilogue, pruner."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
for (M, N, K, V, opts) in ((2048, 128, 2048, 64, {}), (1024, 1024, 512, 64, {"persistent": 2}),
                           (1024, 256, 2048, 64, {"split": 4, "split_mode": 1})):
    for k, v in opts.items():
        sb.set_option(k, v)
    mask = torch.from_numpy(bench.synth_mask(M, K, V, K // 4, 1234)).to(dev)
    a = sb.compress_shflbw(bench.uniform16(torch, (M, K), 1, dev), mask, V)
    B = bench.uniform16(torch, (K, N), 2, dev)
    c = sb.spmm_execute(a, B, out_dtype=torch.bfloat16)
    outs = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(2)]
    sb.spmm_groups_peers(a, 0, a.group_count(), B, outs)
    for k in opts:
        sb.set_option(k, 0)
for (C, H, Kf) in ((16, 8, 64), (16, 7, 64)):
    crs = C * 9
    mask = torch.from_numpy(bench.synth_mask(Kf, crs, 64, crs // 4, 1234)).to(dev)
    w = sb.compress_shflbw(bench.uniform16(torch, (Kf, crs), 3, dev), mask, 64)
    x = bench.uniform16(torch, (C, H, H, 32), 4, dev)
    geo = sb.ConvGeometry(3, 3, 1, 1)
    y1 = sb.conv2d(w, x, geo)
    y2 = sb.conv2d(sb.conv_prepare(w, geo), x, geo)
torch.cuda.synchronize()
print("sanitize smoke ok")
