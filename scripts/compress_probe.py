"""Converter (compress_shflbw) timing (development): wall and device time per
call, warm allocator, north-star and large-FFN shapes."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
for name, M, K, V in (("ns", 2048, 2048, 64), ("lf", 16384, 4096, 64), ("ffn1", 2048, 512, 64)):
    mask = torch.from_numpy(bench.synth_mask(M, K, V, K // 4, 1234)).to(dev)
    W = bench.uniform16(torch, (M, K), 100, dev)
    for _ in range(3):
        a = sb.compress_shflbw(W, mask, V)
        del a
    torch.cuda.synchronize()
    walls, gpus = [], []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record()
        a = sb.compress_shflbw(W, mask, V)
        e1.record()
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t) * 1e3)
        gpus.append(e0.elapsed_time(e1))
        del a
    walls.sort(), gpus.sort()
    print(json.dumps({"shape": name, "M": M, "K": K, "wall_ms_median": round(walls[5], 3),
                      "event_ms_median": round(gpus[5], 3), "wall_ms_min": round(walls[0], 3)}), flush=True)

# asynchronous converter (no host sync): enqueue wall time and device time,
# converting into the same bound-sized matrix (the captured-graph use)
for name, M, K, V in (("ns", 2048, 2048, 64), ("lf", 16384, 4096, 64), ("ffn1", 2048, 512, 64)):
    mask = torch.from_numpy(bench.synth_mask(M, K, V, K // 4, 1234)).to(dev)
    W = bench.uniform16(torch, (M, K), 100, dev)
    a, st = sb.compress_shflbw_async(W, mask, V)
    for _ in range(3):
        sb.compress_shflbw_async(W, mask, V, out=a, status=st)
    torch.cuda.synchronize()
    enq, gpus = [], []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t = time.perf_counter()
        sb.compress_shflbw_async(W, mask, V, out=a, status=st)
        enq.append((time.perf_counter() - t) * 1e3)
        e1.record()
        torch.cuda.synchronize()
        gpus.append(e0.elapsed_time(e1))
    # the same pipeline as one CUDA graph replay
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sb.compress_shflbw_async(W, mask, V, out=a, status=st)
    g.replay()
    torch.cuda.synchronize()
    gr = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        gr.append(e0.elapsed_time(e1))
    sb.finalize(a, st)
    enq.sort(), gpus.sort(), gr.sort()
    print(json.dumps({"async_shape": name, "M": M, "K": K, "enqueue_ms_median": round(enq[5], 3),
                      "event_ms_median": round(gpus[5], 3), "graph_replay_ms_median": round(gr[5], 3)}),
          flush=True)

# allocation check: repeated compress + free must not grow device usage
mask = torch.from_numpy(bench.synth_mask(2048, 2048, 64, 512, 1234)).to(dev)
W = bench.uniform16(torch, (2048, 2048), 100, dev)
for _ in range(5):
    del_a = sb.compress_shflbw(W, mask, 64)
    del del_a
torch.cuda.synchronize()
f0 = torch.cuda.mem_get_info()[0]
for _ in range(200):
    a = sb.compress_shflbw(W, mask, 64)
    del a
torch.cuda.synchronize()
f1 = torch.cuda.mem_get_info()[0]
print(json.dumps({"free_mb_before": f0 // 2**20, "free_mb_after_200": f1 // 2**20}), flush=True)
