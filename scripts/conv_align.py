"""Conv activation-segment alignment probe (development): a 3x1 filter
(s = 0 for every tap) with pad 0 (segments at q0*Nb: 128-byte aligned) vs
pad 1 (segments at (q0-1)*Nb: 64 bytes off), same output grid and K."""
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
C, Kf, Nb, V = 128, 64, 32, 64
for name, H, W, pad in (("aligned pad0", 58, 56, 0), ("misaligned pad1", 56, 54, 1)):
    crs = C * 3
    mask = torch.from_numpy(bench.synth_mask(Kf, crs, V, crs // 4, 1234)).to(dev)
    n = 8
    ws = [sb.conv_prepare(sb.compress_shflbw(bench.uniform16(torch, (Kf, crs), 100 + s, dev), mask, V), 1)
          for s in range(n)]
    xs = [bench.uniform16(torch, (C, H, W, Nb), 300 + s, dev) for s in range(n)]
    P, Q = H + 2 * pad - 3 + 1, W + 2 * pad - 1 + 1
    outs = [torch.empty((Kf, P, Q, Nb), dtype=torch.bfloat16, device=dev) for _ in range(n)]
    lib = sb.shflbw._lib()

    def step(i):
        k = i % n
        assert lib.shflbw_cu_conv2d(ws[k].ptr, xs[k].data_ptr(), C, H, W, Nb, 3, 1, 1, pad, outs[k].data_ptr(),
                                    1, torch.cuda.current_stream().cuda_stream) == 0
    for opt in (-1, 2):
        sb.set_option("persistent", opt)
        us = sweep.time_steps(step, 300) * 1e3
        print(json.dumps({"case": name, "P": P, "Q": Q, "persistent": opt, "us": round(us, 2)}), flush=True)
    sb.set_option("persistent", 0)
