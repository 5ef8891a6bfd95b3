"""Development: per-CTA timelines of two consecutive SpMM launches in a PDL
chain (trace build), on one clock: when the successor's CTAs enter relative
to the predecessor's events."""
import argparse
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="ns")
ap.add_argument("--opts", default="")
ap.add_argument("--chain", type=int, default=8)
args = ap.parse_args()
wl = dict(bench.WORKLOADS[args.workload])
M, N, K, V, alpha = wl["M"], wl["N"], wl["K"], wl["V"], wl["alpha"]
dev = torch.device("cuda", 0)
mask = torch.from_numpy(bench.synth_mask(M, K, V, int(round(alpha * K)), 1234)).to(dev)
nset = args.chain
mats = [sb.compress_shflbw(bench.uniform16(torch, (M, K), 100 + i, dev), mask, V) for i in range(nset)]
Bs = [bench.uniform16(torch, (K, N), 200 + i, dev) for i in range(nset)]
Cs = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for i in range(nset)]
for kv in [x for x in args.opts.split(",") if x]:
    k, v = kv.split("=")
    sb.set_option(k, int(v))
trA = torch.zeros(1 << 20, dtype=torch.int64, device=dev)
trB = torch.zeros(1 << 20, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
names = ["entry", "setup", "dep_wait", "first_full", "last_mma", "accum", "epi_done", "exit"]
extra = {24: "partial_ok", 25: "recv_ok", 26: "sum_done", 27: "tile_bar", 28: "stores_issued",
         16: "issue[0]", 8: "full[0]", 9: "full[1]", 10: "full[2]", 11: "full[3]"}
# the chain is captured in a CUDA graph so the launches run back to back (an
# eager Python loop issues one launch per ~10 us: every launch ran isolated)
s = torch.cuda.Stream()
for i in range(args.chain):  # warm-up (module load, plans)
    sb.spmm_execute(mats[i % nset], Bs[i % nset], out=Cs[i % nset])
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for i in range(args.chain):
        sb.set_option("trace", trA.data_ptr() if i == args.chain - 2 else (trB.data_ptr() if i == args.chain - 1 else 0))
        sb.spmm_execute(mats[i % nset], Bs[i % nset], out=Cs[i % nset])
sb.set_option("trace", 0)
for it in range(3):
    flush.fill_(it)
    torch.cuda.synchronize()
    trA.zero_()
    trB.zero_()
    g.replay()
    torch.cuda.synchronize()
a = trA.cpu().numpy().reshape(-1, 32)
b = trB.cpu().numpy().reshape(-1, 32)
a = a[a[:, 0] > 0]
b = b[b[:, 0] > 0]
t0 = a[:, 0].min()
print(f"{args.workload} {args.opts}: predecessor {len(a)} CTAs, successor {len(b)} CTAs (us after the predecessor's first entry)")
for nm, e in list(zip(names, range(8))) + [(v, k) for k, v in sorted(extra.items())]:
    ca, cb = (a[:, e] - t0) / 1e3, (b[:, e] - t0) / 1e3
    ca, cb = ca[a[:, e] > 0], cb[b[:, e] > 0]
    if not len(ca) or not len(cb):
        continue
    print(f"  {nm:10s} pred min {ca.min():6.2f} p50 {np.median(ca):6.2f} max {ca.max():6.2f} | "
          f"succ min {cb.min():6.2f} p50 {np.median(cb):6.2f} max {cb.max():6.2f}")
