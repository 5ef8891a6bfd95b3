"""the paper's format comparison on B200.

    python scripts/compare_formats.py [--out profiles/formats_r1]

For each shape and density, times (bench protocol: rotating L2-defeating
input sets, CUDA graph, CUDA events):
  * Shfl-BW: V-row groups of arbitrary (shuffled) rows -- the write-back goes
    through row_indices;
  * VW (vector-wise): the same kernel on a mask whose groups are V
    consecutive rows, so row_indices is the identity (the paper's "row
    shuffling is nearly free" claim, is Shfl-BW / VW ~ 1);
  * BW (block-wise V x V, the same density) through this library: every K
    block is one contiguous 64-column run, loaded as two TMA 2D tiles (and,
    for comparison, with the Shfl-BW gathers); and through the library BSR
    kernel (torch.sparse_bsr_tensor @ dense, cuSPARSE), where it runs;
  * dense cuBLAS bf16 GEMM.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402
import sweep  # noqa: E402

SHAPES = [("north star", 2048, 128, 2048, 64), ("GNMT", 4096, 128, 1024, 64),
          ("FFN2 N=4096", 512, 4096, 2048, 64), ("FFN1 N=4096", 2048, 4096, 512, 64)]


def vw_mask(M, K, V, cpg, seed):
    """Vector-wise: groups of V consecutive rows share a random column set."""
    rs = np.random.RandomState(seed)
    G = M // V
    cols = np.argsort(rs.rand(G, K), axis=1)[:, :cpg]
    vw = np.zeros((G, K), np.uint8)
    np.put_along_axis(vw, cols, 1, axis=1)
    return np.repeat(vw, V, axis=0)


def bw_mask(M, K, V, alpha, seed):
    """Block-wise V x V blocks, each block row keeping round(alpha * K/V) blocks."""
    rs = np.random.RandomState(seed)
    kb = K // V
    keep = max(1, int(round(alpha * kb)))
    blocks = np.zeros((M // V, kb), np.uint8)
    for i in range(M // V):
        blocks[i, rs.permutation(kb)[:keep]] = 1
    return np.kron(blocks, np.ones((V, V), np.uint8))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "formats"))
    ap.add_argument("--steps", type=int, default=300)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rows = []
    for name, M, N, K, V in SHAPES:
        for alpha in (0.25, 0.1):
            cpg = int(round(alpha * K))
            set_bytes = 2 * M * cpg + 2 * K * N + 2 * M * N
            n = 1 if set_bytes > bench.L2_BYTES else min(64, max(2, math.ceil(1.25 * bench.L2_BYTES / set_bytes)))
            Bs = [bench.uniform16(torch, (K, N), 200 + s, dev) for s in range(n)]
            Cs = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(n)]
            Ws = [bench.uniform16(torch, (M, K), 100 + s, dev) for s in range(n)]
            res = {"shape": name, "M": M, "N": N, "K": K, "V": V, "sparsity": 1 - alpha}
            for fmt, mk in (("shflbw", lambda: bench.synth_mask(M, K, V, cpg, 1234)),
                            ("vw", lambda: vw_mask(M, K, V, cpg, 1234))):
                mask = torch.from_numpy(mk()).to(dev)
                mats = [sb.compress_shflbw(w, mask, V) for w in Ws]
                res[fmt + "_us"] = sweep.time_steps(lambda i: sb.spmm_execute(mats[i % n], Bs[i % n], out=Cs[i % n]),
                                                    args.steps) * 1e3
            res["shflbw_over_vw"] = res["shflbw_us"] / res["vw_us"]
            res["dense_us"] = sweep.time_steps(lambda i: torch.mm(Ws[i % n], Bs[i % n], out=Cs[i % n]),
                                               args.steps) * 1e3
            # block-wise V x V through this library: every K block is one
            # contiguous 64-column run -> two TMA 2D tiles per K block (default)
            # or, for comparison, the same gathers as Shfl-BW
            bwm = torch.from_numpy(bw_mask(M, K, V, alpha, 1234)).to(dev)
            bmats = [sb.compress_shflbw(w, bwm, V) for w in Ws]
            for tl, key in ((0, "bw_tiles_us"), (-1, "bw_gathers_us")):
                sb.set_option("tile_loads", tl)
                res[key] = sweep.time_steps(lambda i: sb.spmm_execute(bmats[i % n], Bs[i % n], out=Cs[i % n]),
                                            args.steps) * 1e3
            sb.set_option("tile_loads", 0)
            res["shflbw_over_bw"] = res["shflbw_us"] / res["bw_tiles_us"]
            try:  # block-wise through the library BSR kernel (cuSPARSE)
                bm = torch.from_numpy(bw_mask(M, K, V, alpha, 1234)).to(dev).to(torch.bfloat16)
                bsr = [(w * bm).to_sparse_bsr((V, V)) for w in Ws]
                res["bsr_us"] = sweep.time_steps(lambda i: torch.matmul(bsr[i % n], Bs[i % n]), args.steps) * 1e3
            except Exception as e:  # noqa: BLE001
                res["bsr_us"] = None
                res["bsr_error"] = f"{type(e).__name__}: {str(e)[:120]}"
            rows.append(res)
            print(json.dumps(res), flush=True)
    lines = ["| shape | sparsity | Shfl-BW us | VW us | Shfl-BW / VW | BW us (TMA tiles) | BW us (gathers) | "
             "Shfl-BW / BW | BW via cuSPARSE BSR us | dense cuBLAS us |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        bsr = f"{r['bsr_us']:.2f}" if r["bsr_us"] else "n/a"
        lines.append(f"| {r['shape']} | {r['sparsity']:.0%} | {r['shflbw_us']:.2f} | {r['vw_us']:.2f} | "
                     f"{r['shflbw_over_vw']:.3f} | {r['bw_tiles_us']:.2f} | {r['bw_gathers_us']:.2f} | "
                     f"{r['shflbw_over_bw']:.3f} | {bsr} | {r['dense_us']:.2f} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(args.out + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
