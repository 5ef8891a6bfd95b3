"""GPU prune_shflbw vs the compiled reference (oracle/_ref, single-threaded
like the reference's pruner) on synthetic importance scores; checks the
results are identical."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_05016_b200 as sb  # noqa: E402
from oracle import Reference  # noqa: E402

ref = Reference()
for (M, K, V, alpha, iters, restarts) in ((512, 512, 32, 0.25, 20, 2), (1024, 1024, 32, 0.25, 20, 2),
                                          (2048, 2048, 64, 0.25, 20, 1)):
    s = np.abs(ref.random_dense(M, K, 1)).astype(np.float32)
    cfg = {"alpha": alpha, "beta_factor": 2.0, "v": V, "kmeans_max_iters": iters, "seed": 0, "restarts": restarts}
    t0 = time.perf_counter()
    mask, perm, kept = ref.prune_shflbw(s, cfg)
    t_ref = time.perf_counter() - t0
    sd = torch.from_numpy(s).cuda()
    sb.prune_shflbw(sd, sb.PruneConfig(**cfg))  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = sb.prune_shflbw(sd, sb.PruneConfig(**cfg))
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    same = (np.array_equal(r.mask.cpu().numpy(), mask) and
            np.array_equal(r.permutation.cpu().numpy().astype(np.uint32), perm) and
            float(r.kept_score).hex() == float(kept).hex())
    print(json.dumps({"M": M, "K": K, "V": V, "alpha": alpha, "kmeans_max_iters": iters, "restarts": restarts,
                      "reference_s": round(t_ref, 3), "gpu_s": round(t_gpu, 4), "speedup": round(t_ref / t_gpu, 1),
                      "identical": bool(same)}), flush=True)
