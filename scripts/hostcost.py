"""Host-side cost of one SpMM call through the public API (development tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ctypes as C
import torch
import bench
import paper_2203_05016_b200 as sb
from paper_2203_05016_b200 import _lib as L

dev = torch.device("cuda", 0)
M, N, K, V = 2048, 128, 2048, 64
mask = torch.from_numpy(bench.synth_mask(M, K, V, 512, 1)).to(dev)
a = sb.compress_shflbw(bench.uniform16(torch, (M, K), 1, dev), mask, V)
B = bench.uniform16(torch, (K, N), 2, dev)
Cc = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
lib = L.load()
s = torch.cuda.current_stream().cuda_stream
for name, fn in [("python spmm_execute", lambda: sb.spmm_execute(a, B, out=Cc)),
                 ("raw ctypes shflbw_cu_spmm", lambda: lib.shflbw_cu_spmm(a.ptr, B.data_ptr(), K, N, N, Cc.data_ptr(), 1, N, s)),
                 ("torch.mm dense (cuBLAS)", None)]:
    if fn is None:
        Wd = sb.decompress(a).to(torch.bfloat16)
        fn = lambda: torch.mm(Wd, B, out=Cc)
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    n = 2000
    for _ in range(n):
        fn()
    el = time.perf_counter() - t
    torch.cuda.synchronize()
    print(f"{name:28s} {el / n * 1e6:7.2f} us host per call")
