"""Per-CTA event timeline of one SpMM launch (development tool).

Events (globaltimer ns): 0 entry, 1 setup done, 2 grid-dependency wait
returned, 3 first stage full (MMA), 4 last MMA issued, 5 accumulator ready,
6 epilogue stores done, 7 exit.  Prints percentiles relative to the
earliest CTA entry.
"""
import argparse, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2203_05016_b200 as sb

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="ns")
ap.add_argument("--opts", default="")
ap.add_argument("--K", type=int, default=0)
ap.add_argument("--chain", type=int, default=0, help="launch this many SpMMs back to back on rotating "
                "operand sets (warm, PDL-overlapped) and trace the last one")
ap.add_argument("--persist", action="store_true", help="print the persistent kernel's per-unit events")
args = ap.parse_args()
wl = dict(bench.WORKLOADS[args.workload])
if args.K:
    wl["K"] = args.K
M, N, K, V, alpha = wl["M"], wl["N"], wl["K"], wl["V"], wl["alpha"]
dev = torch.device("cuda", 0)
cpg = int(round(alpha * K))
mask = torch.from_numpy(bench.synth_mask(M, K, V, cpg, 1234)).to(dev)
nset = max(1, args.chain)
if os.environ.get("SBW_WARM"):  # development: one L2-resident operand set, reused by every launch
    nset = 1
mats = [sb.compress_shflbw(bench.uniform16(torch, (M, K), 100 + i, dev), mask, V) for i in range(nset)]
Bs = [bench.uniform16(torch, (K, N), 200 + i, dev) for i in range(nset)]
Cs = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for i in range(nset)]
a, B, C = mats[0], Bs[0], Cs[0]
for kv in [x for x in args.opts.split(",") if x]:
    k, v = kv.split("=")
    sb.set_option(k, int(v))
tr = torch.zeros(1 << 20, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for it in range(3):
    if not os.environ.get("SBW_WARM"):
        flush.fill_(it)  # cold L2
    torch.cuda.synchronize()
    tr.zero_()
    sb.set_option("trace", tr.data_ptr())
    if args.chain:
        for i in range(args.chain):
            sb.spmm_execute(mats[i % nset], Bs[i % nset], out=Cs[i % nset])
    else:
        sb.spmm_execute(a, B, out=C)
    torch.cuda.synchronize()
    sb.set_option("trace", 0)
t = tr.cpu().numpy().reshape(-1, 32)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
names = ["entry", "setup", "dep_wait", "first_full", "last_mma", "accum", "epi_done", "exit"]
names += [f"full[{k}]" for k in range(8)] + [f"issue[{k}]" for k in range(8)] + ["partial_ok", "recv_ok",
          "sum_done", "tile_bar", "stores_issued", "mma_done[0]", "mma_done[1]", "mma_done[2]"]
print(f"{args.workload} K={K} {args.opts} chain={args.chain}: {len(t)} CTAs, span {rel[:, 7].max():.2f} us, "
      f"dep_wait(min)->exit(max) {rel[:, 7].max() - rel[t[:, 2] > 0, 2].min():.2f} us")
for e, nm in enumerate(names):
    if not nm:
        continue
    col = rel[:, e]
    col = col[t[:, e] > 0]
    if len(col):
        print(f"  {nm:10s} min {col.min():7.2f}  p50 {np.median(col):7.2f}  max {col.max():7.2f} us")

if args.persist:
    dep = rel[:, 2]
    print("  per unit i (median over CTAs, us after the CTA's dependency wait): gathers start / MMA start / "
          "accumulated")
    for i in range(8):
        cols = [rel[:, 16 + i] - dep, rel[:, 8 + i] - dep, rel[:, 24 + i] - dep]
        ok = t[:, 24 + i] > 0
        if ok.sum() == 0:
            break
        print(f"  unit {i}: " + "  ".join(f"{np.median(c[ok]):7.2f}" for c in cols))
