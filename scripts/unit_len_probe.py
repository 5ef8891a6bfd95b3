"""Unit-length probe (development): SpMMs with the same total gather work
(units x K blocks) but different K blocks per unit, dense masks (alpha = 1)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import paper_2203_05016_b200 as sb  # noqa: E402
import sweep  # noqa: E402

dev = torch.device("cuda", 0)
opts = [x for x in (sys.argv[1] if len(sys.argv) > 1 else "").split(";")]
for o in opts:
    for kv in [x for x in o.split(",") if x]:
        k, v = kv.split("=")
        sb.set_option(k, int(v))
    for (M, N, K) in ((64, 100352, 192), (64, 50176, 384), (64, 25088, 768), (64, 12544, 1536), (64, 6272, 3072),
                      (256, 25088, 192), (256, 6272, 768)):
        r = sweep.spmm_row("u", M, N, K, 64, 1.0, 300, dev)
        print(json.dumps({"opts": o, "M": M, "N": N, "K": K, "kb_per_unit": K // 64, "units": (M // 64) * (N // 128),
                          "us": round(r["us"], 2), "dense_us": round(r["dense_us"], 2)}), flush=True)
    for kv in [x for x in o.split(",") if x]:
        sb.set_option(kv.split("=")[0], 0)
