"""Conv vs SpMM probe (development): the ResNet 3x3 @56 conv against an SpMM
with the same unit structure (1 group of V=64, 3 K blocks, 784 column tiles),
under several launch options.  Separates the conv addressing from the
pipeline structure.

    python scripts/conv_probe.py [--configs "persistent=-1;persistent=2,stages=2"]
"""
import argparse
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

DEFAULTS = {"split": 0, "pdl": 1, "stages": 0, "persistent": 0, "split_mode": 0}


def with_opts(cfg, fn):
    opts = dict(DEFAULTS)
    for kv in [x for x in cfg.split(",") if x]:
        k, v = kv.split("=")
        opts[k] = int(v)
    for k, v in opts.items():
        sb.set_option(k, v)
    try:
        return fn()
    finally:
        for k, v in DEFAULTS.items():
            sb.set_option(k, v)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="persistent=0;persistent=-1;persistent=1;persistent=2,stages=2")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--convs", default="56,28,14,7")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = sb.shflbw._lib()
    table = {56: (64, 64), 28: (128, 128), 14: (256, 256), 7: (512, 512)}
    for H in [int(x) for x in args.convs.split(",")]:
        C, Kf = table[H]
        R, pad, Nb, V = 3, 1, 32, 64
        crs = C * R * R
        mask = torch.from_numpy(bench.synth_mask(Kf, crs, V, crs // 4, 1234)).to(dev)
        geo = sb.ConvGeometry(R, R, 1, pad)
        n = 6
        ws = [sb.conv_prepare(sb.compress_shflbw(bench.uniform16(torch, (Kf, crs), 100 + s, dev), mask, V), geo)
              for s in range(n)]
        xs = [bench.uniform16(torch, (C, H, H, Nb), 300 + s, dev) for s in range(n)]
        outs = [torch.empty((Kf, H, H, Nb), dtype=torch.bfloat16, device=dev) for _ in range(n)]

        def conv_step(i):
            k = i % n
            assert lib.shflbw_cu_conv2d(ws[k].ptr, xs[k].data_ptr(), C, H, H, Nb, R, R, 1, pad, outs[k].data_ptr(),
                                        1, torch.cuda.current_stream().cuda_stream) == 0

        # SpMM with the same units: M = Kf, K' = the conv's padded group width
        kp = ws[0].total_cols // max(1, ws[0].group_count())
        N = H * H * Nb
        K = kp
        smask = torch.ones((Kf, K), dtype=torch.uint8, device=dev)
        mats = [sb.compress_shflbw(bench.uniform16(torch, (Kf, K), 100 + s, dev), smask, V) for s in range(n)]
        Bs = [bench.uniform16(torch, (K, N), 200 + s, dev) for s in range(n)]
        Cs = [torch.empty((Kf, N), dtype=torch.bfloat16, device=dev) for _ in range(n)]

        def spmm_step(i):
            k = i % n
            sb.spmm_execute(mats[k], Bs[k], out=Cs[k])

        for cfg in [c for c in args.configs.split(";")]:
            t_conv = with_opts(cfg, lambda: sweep.time_steps(conv_step, args.steps)) * 1e3
            t_spmm = with_opts(cfg, lambda: sweep.time_steps(spmm_step, args.steps)) * 1e3
            print(json.dumps({"conv": f"3x3 {C}@{H}", "cfg": cfg, "conv_us": round(t_conv, 2),
                              "spmm_same_units_us": round(t_spmm, 2), "kp": kp, "N": N}), flush=True)


if __name__ == "__main__":
    main()
