"""Kernel-option sweep on one GPU (development tool, not the bench).

    python scripts/explore.py [--workload ns] [--steps 2000]

Times the SpMM under several launch options (V split, stages, PDL,
CUDA-core path) with the bench protocol (rotating L2-defeating sets, CUDA
graph, events) and prints one line per option set.
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="ns")
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--configs", default="")
    ap.add_argument("--M", type=int, default=0)
    ap.add_argument("--N", type=int, default=0)
    ap.add_argument("--K", type=int, default=0)
    ap.add_argument("--V", type=int, default=0)
    args = ap.parse_args()
    wl = dict(bench.WORKLOADS[args.workload])
    for k in "MNKV":
        if getattr(args, k):
            wl[k] = getattr(args, k)
    M, N, K, V, alpha = wl["M"], wl["N"], wl["K"], wl["V"], wl["alpha"]
    dev = torch.device("cuda", 0)
    cpg = int(round(alpha * K))
    mask = torch.from_numpy(bench.synth_mask(M, K, V, cpg, 1234)).to(dev)
    kpad = (cpg + 63) // 64 * 64
    set_bytes = 2 * M * kpad + 4 * (M // V) * kpad + 2 * K * N + 2 * M * N
    nsets = 1 if set_bytes > bench.L2_BYTES else min(64, max(2, math.ceil(1.25 * bench.L2_BYTES / set_bytes)))
    mats = [sb.compress_shflbw(bench.uniform16(torch, (M, K), 100 + s, dev), mask, V) for s in range(nsets)]
    Bs = [bench.uniform16(torch, (K, N), 200 + s, dev) for s in range(nsets)]
    Cs = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(nsets)]

    def step(i):
        s = i % nsets
        sb.spmm_execute(mats[s], Bs[s], out=Cs[s])

    configs = [c for c in args.configs.split(";") if c] or [
        "split=1", "split=2", "split=4", "split=0,pdl=0", "split=0",
        "split=1,cp_async_slabs=1", "split=1,cp_async_slabs=2",
        "split=1,cp_async_slabs=1,stages=6", "split=1,cp_async_slabs=2,stages=6",
        "split=0,stages=2", "split=0,stages=6"]
    print(f"workload M={M} N={N} K={K} V={V} alpha={alpha} sets={nsets}")
    for cfg in configs:
        opts = {"split": 0, "pdl": 1, "stages": 0, "force_simt": 0, "cp_async_slabs": 0, "split_mode": 0, "persistent": 0}
        for kv in cfg.split(","):
            k, v = kv.split("=")
            opts[k] = int(v)
        for k, v in opts.items():
            sb.set_option(k, v)
        ms, _, _ = bench.graph_time(torch, step, args.steps, 50, 0.1, lambda: None)
        us = ms / args.steps * 1e3
        print(f"{cfg:32s} {us:8.2f} us/step  {2 * M * N * K / (us * 1e-6) / 1e12:8.1f} dense-eq TFLOP/s",
              flush=True)
    for k, v in {"split": 0, "pdl": 1, "stages": 0, "force_simt": 0, "cp_async_slabs": 0, "split_mode": 0, "persistent": 0}.items():
        sb.set_option(k, v)


if __name__ == "__main__":
    main()
