"""Conv row-size probe: the same 3x3 convs at batch 32 (64-byte gather rows)
and batch 64 (128-byte rows)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import sweep  # noqa: E402

dev = torch.device("cuda", 0)
for C, H in ((64, 56), (128, 28), (256, 14)):
    for Nb in (16, 32, 64):
        r = sweep.conv_row(f"3x3 {C}@{H} Nb={Nb}", C, H, C, 3, 1, Nb, 64, 0.25, 200, dev)
        print(json.dumps({k: r[k] for k in ("name", "us", "dense_us", "speedup", "rel_err_vs_cudnn_bf16")}), flush=True)
