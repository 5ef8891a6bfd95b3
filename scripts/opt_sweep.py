"""Time selected BASELINE sweep configurations under several option sets.

    python scripts/opt_sweep.py --opts "persistent=-1;persistent=1" --only "FFN1,ResNet 3x3"
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import paper_2203_05016_b200 as sb  # noqa: E402
import sweep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--opts", default="persistent=-1;persistent=1")
ap.add_argument("--only", default="")
ap.add_argument("--steps", type=int, default=200)
args = ap.parse_args()
dev = torch.device("cuda", 0)
keys = [k for k in args.only.split(",") if k]
for cfg in sweep.SPMM + sweep.CONV:
    if keys and not any(k in cfg[0] for k in keys):
        continue
    line = {"name": cfg[0]}
    for o in [x for x in args.opts.split(";") if x]:
        for kv in o.split(","):
            k, v = kv.split("=")
            sb.set_option(k, int(v))
        if cfg in sweep.SPMM:
            r = sweep.spmm_row(*cfg, args.steps if cfg[1] * cfg[2] < 1 << 26 else 20, dev)
        else:
            r = sweep.conv_row(*cfg, args.steps, dev)
        line[o] = round(r["us"], 2)
        line["dense"] = round(r["dense_us"], 2)
        for kv in o.split(","):
            sb.set_option(kv.split("=")[0], 0)
    print(json.dumps(line), flush=True)
