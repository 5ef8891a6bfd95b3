"""Per-CTA event timeline of sparse implicit-GEMM conv launches (development
tool; needs an SBW_TRACE build, see scripts/trace.py).

    python scripts/conv_trace.py --workload conv56 [--chain 8] [--opts k=v,...]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402

CONV = {"conv56": (64, 56, 64, 3, 1, 32, 64, 0.25), "conv28": (128, 28, 128, 3, 1, 32, 64, 0.25),
        "conv14": (256, 14, 256, 3, 1, 32, 64, 0.25), "conv7": (512, 7, 512, 3, 1, 32, 64, 0.25)}
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="conv56")
ap.add_argument("--opts", default="")
ap.add_argument("--chain", type=int, default=4)
ap.add_argument("--prepared", action="store_true")
ap.add_argument("--persist", action="store_true")
args = ap.parse_args()

C, H, Kf, R, pad, Nb, V, alpha = CONV[args.workload]
dev = torch.device("cuda", 0)
crs = C * R * R
mask = torch.from_numpy(bench.synth_mask(Kf, crs, V, int(round(alpha * crs)), 1234)).to(dev)
nset = max(1, args.chain)
ws = [sb.compress_shflbw(bench.uniform16(torch, (Kf, crs), 100 + i, dev), mask, V) for i in range(nset)]
if args.prepared:
    ws = [sb.conv_prepare(w, R) for w in ws]
xs = [bench.uniform16(torch, (C, H, H, Nb), 300 + i, dev) for i in range(nset)]
P = H + 2 * pad - R + 1
outs = [torch.empty((Kf, P, P, Nb), dtype=torch.bfloat16, device=dev) for _ in range(nset)]
for kv in [x for x in args.opts.split(",") if x]:
    k, v = kv.split("=")
    sb.set_option(k, int(v))
lib = sb.shflbw._lib()
tr = torch.zeros(1 << 22, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
for it in range(3):
    flush.fill_(it)
    torch.cuda.synchronize()
    tr.zero_()
    sb.set_option("trace", tr.data_ptr())
    for i in range(nset):
        assert lib.shflbw_cu_conv2d(ws[i].ptr, xs[i].data_ptr(), C, H, H, Nb, R, R, 1, pad, outs[i].data_ptr(), 1, st) == 0
    torch.cuda.synchronize()
    sb.set_option("trace", 0)
t = tr.cpu().numpy().reshape(-1, 32)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
names = ["entry", "setup", "dep_wait", "first_full", "last_mma", "accum", "epi_done", "exit"]
names += [f"full[{k}]" for k in range(8)] + [f"issue[{k}]" for k in range(8)]
print(f"{args.workload} {args.opts} chain={args.chain}: {len(t)} CTAs, span {rel[:, 7].max():.2f} us")
for e, nm in enumerate(names):
    col = rel[:, e][t[:, e] > 0]
    if len(col):
        print(f"  {nm:10s} min {col.min():7.2f}  p10 {np.percentile(col, 10):7.2f}  p50 {np.median(col):7.2f}  "
              f"p90 {np.percentile(col, 90):7.2f}  max {col.max():7.2f} us")
# per-CTA durations
d = rel[:, 7] - rel[:, 0]
print(f"  CTA lifetime p50 {np.median(d):.2f} us, max {d.max():.2f}; first_full-dep {np.median(rel[:, 3] - rel[:, 2]):.2f}; "
      f"full[k+1]-full[k] p50 {np.median(rel[:, 9] - rel[:, 8]):.2f}; accum->exit p50 {np.median(rel[:, 7] - rel[:, 5]):.2f}")

if args.persist:
    dep = rel[:, 2]
    print("  per unit i (median over CTAs, us after the CTA's dependency wait): gathers start / MMA start / "
          "accumulated")
    for i in range(8):
        ok = t[:, 24 + i] > 0
        if ok.sum() == 0:
            break
        cols = [rel[:, 16 + i] - dep, rel[:, 8 + i] - dep, rel[:, 24 + i] - dep]
        print(f"  unit {i}: " + "  ".join(f"{np.median(c[ok]):7.2f}" for c in cols) + f"   ({ok.sum()} CTAs)")
