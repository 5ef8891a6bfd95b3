"""Conv / SpMM cold-vs-warm input probe (development): the same launch with
1 input set (stays in L2) vs 12 rotating sets (cold every step)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402
import sweep  # noqa: E402

dev = torch.device("cuda", 0)
lib = sb.shflbw._lib()
for (C, H, Kf) in ((64, 56, 64), (128, 28, 128), (256, 14, 256)):
    R, pad, Nb, V = 3, 1, 32, 64
    crs = C * R * R
    mask = torch.from_numpy(bench.synth_mask(Kf, crs, V, crs // 4, 1234)).to(dev)
    geo = sb.ConvGeometry(R, R, 1, pad)
    for n in (1, 12):
        ws = [sb.conv_prepare(sb.compress_shflbw(bench.uniform16(torch, (Kf, crs), 100 + s, dev), mask, V), geo)
              for s in range(n)]
        xs = [bench.uniform16(torch, (C, H, H, Nb), 300 + s, dev) for s in range(n)]
        outs = [torch.empty((Kf, H, H, Nb), dtype=torch.bfloat16, device=dev) for _ in range(n)]

        def step(i):
            k = i % n
            assert lib.shflbw_cu_conv2d(ws[k].ptr, xs[k].data_ptr(), C, H, H, Nb, R, R, 1, pad, outs[k].data_ptr(),
                                        1, torch.cuda.current_stream().cuda_stream) == 0
        us = sweep.time_steps(step, 300) * 1e3
        print(json.dumps({"conv": f"3x3 {C}@{H}", "sets": n, "us": round(us, 2)}), flush=True)
for name, M, N, K in (("FFN2", 512, 4096, 2048), ("FFN1", 2048, 4096, 512)):
    V = 64
    mask = torch.from_numpy(bench.synth_mask(M, K, V, K // 4, 1234)).to(dev)
    for n in (1, 12):
        mats = [sb.compress_shflbw(bench.uniform16(torch, (M, K), 100 + s, dev), mask, V) for s in range(n)]
        Bs = [bench.uniform16(torch, (K, N), 200 + s, dev) for s in range(n)]
        Cs = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(n)]
        us = sweep.time_steps(lambda i: sb.spmm_execute(mats[i % n], Bs[i % n], out=Cs[i % n]), 300) * 1e3
        print(json.dumps({"spmm": name, "sets": n, "us": round(us, 2)}), flush=True)
