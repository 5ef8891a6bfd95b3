"""PCIe copy probe (development): pinned 512 KB H2D / D2H alone and concurrent."""
import torch
from cuda.bindings import runtime as rt

n = 512 * 1024
hb = torch.empty(n, dtype=torch.uint8).pin_memory()
hc = torch.empty(n, dtype=torch.uint8).pin_memory()
db = torch.empty(n, dtype=torch.uint8, device="cuda")
dc = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
H2D, D2H = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost


def timed(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


r1, r2 = rt.cudaStream_t(s1.cuda_stream), rt.cudaStream_t(s2.cuda_stream)
h2d = timed(lambda: rt.cudaMemcpyAsync(db.data_ptr(), hb.data_ptr(), n, H2D, r1))
d2h = timed(lambda: rt.cudaMemcpyAsync(hc.data_ptr(), dc.data_ptr(), n, D2H, r1))
both = timed(lambda: (rt.cudaMemcpyAsync(db.data_ptr(), hb.data_ptr(), n, H2D, r1),
                      rt.cudaMemcpyAsync(hc.data_ptr(), dc.data_ptr(), n, D2H, r2)))
print(f"H2D 512KB {h2d:.2f} us ({n / h2d / 1e3:.1f} GB/s), D2H {d2h:.2f} us ({n / d2h / 1e3:.1f} GB/s), "
      f"concurrent pair {both:.2f} us")
