"""Per-SpMM time in a true layer chain of north-star SpMMs (each consuming
the previous one's bf16 output), as CUDA-graph replays over rotating operand
sets."""
import json
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
M = K = 2048
N, V, L = 128, 64, int(sys.argv[1]) if len(sys.argv) > 1 else 8
nchains = 8  # rotating operand sets (8 chains x 8 matrices x 0.6 MB > L2 with the activations)
mask = torch.from_numpy(bench.synth_mask(M, K, V, K // 4, 1234)).to(dev)
sets = []
for c in range(nchains):
    mats = [sb.compress_shflbw(bench.uniform16(torch, (M, K), 100 + c * L + i, dev), mask, V) for i in range(L)]
    B = bench.uniform16(torch, (K, N), 500 + c, dev)
    outs = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(L)]
    sets.append((mats, B, outs))


def separate(i):
    mats, B, outs = sets[i % nchains]
    x = B
    for a, o in zip(mats, outs):
        sb.spmm_execute(a, x, out_dtype=torch.bfloat16, out=o)
        x = o


res = {}
for name, fn in (("chain_of_separate_calls", separate), ("chain_of_separate_calls", separate)):
    ms, _, _ = bench.graph_time(torch, fn, 200, 10, 0.2, lambda: None)
    res.setdefault(name, []).append(ms / 200 / L * 1e3)
print(json.dumps({"links": L, "us_per_spmm": res}))
