#!/usr/bin/env python
"""bench.py -- Shfl-BW SpMM on B200: dense-equivalent TFLOP/s vs cuBLAS.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload ns|lf|ffn] [--no-cpu-baseline]

Default workload (BASELINE.json north star, configs[0]): Shfl-BW SpMM
M/N/K = 2048/128/2048, V = 64, 75 % sparsity, bf16 operands, fp32
accumulation, bf16 output.  A *step* is one SpMM over one input set (one
kernel launch).  Inputs rotate over enough independent sets (weights,
activations, outputs) that their total exceeds the 126 MB L2, so every step
streams its operands from HBM; the K steps run as CUDA-graph replays and are
timed with CUDA events on the launching stream (max over ranks).

Printed: ONE JSON line (rank 0) with the driver's contract keys plus
`roofline` (dominant kernel vs MEASURED_PEAKS.json), `cpu_baseline` (the
reference's own spmm_execute, compiled from its sources, on this host's
cores), `e2e` (the same metric through the public API with pinned host
buffers and the H2D/D2H copies inside the timed region), `clocks` (NVML,
sampled during the timed region) and the cuBLAS dense bf16 GEMM of the same
shape.

`--impl reference` times the reference's CPU implementation
(oracle/_ref/libshflbw_ref.so: /root/reference/proj/src compiled unmodified)
on the same workload with all host threads; under torchrun only rank 0 runs.

Workloads: ns (default), ffn (Transformer FFN2 512x2048, N=4096, 75 %),
lf (large FFN 16384x4096, N=8192, 75 %, row groups sharded over ranks:
strong scaling, optional NCCL all-gather with --allgather).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: M, N, K, V, density, shards (True = row groups split over ranks)
    "ns": dict(M=2048, N=128, K=2048, V=64, alpha=0.25, sharded=False,
               desc="Shfl-BW SpMM M/N/K=2048/128/2048 V=64 75% sparsity (north star)"),
    "ffn": dict(M=512, N=4096, K=2048, V=64, alpha=0.25, sharded=False,
                desc="Transformer-base FFN2 512x2048, N=4096, V=64, 75% sparsity"),
    "lf": dict(M=16384, N=8192, K=4096, V=64, alpha=0.25, sharded=True,
               desc="Large FFN 16384x4096, N=8192, V=64, 75% sparsity, M-row-group sharded"),
}
METRIC = "dense-equiv TFLOP/s & speedup vs cuBLAS dense GEMM; tensor-pipe util %"
UNIT = "TFLOP/s (dense-equivalent, 2*M*N*K/t)"
L2_BYTES = 126 * 1024 * 1024


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------
# synthetic inputs (SURVEY.md §8(d) shapes; a vector-wise mask with rows
# scattered by a random permutation, U[-1,1) values rounded to bf16)
# --------------------------------------------------------------------------

def synth_mask(M, K, V, cpg, seed):
    rs = np.random.RandomState(seed)
    G = M // V
    cols = np.argsort(rs.rand(G, K), axis=1)[:, :cpg]
    vw = np.zeros((G, K), np.uint8)
    np.put_along_axis(vw, cols, 1, axis=1)
    vw = np.repeat(vw, V, axis=0)
    perm = rs.permutation(M)
    mask = np.empty_like(vw)
    mask[perm] = vw
    return mask


def uniform_bf16(torch, shape, seed, device):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.rand(shape, generator=g, device=device) * 2 - 1).to(torch.bfloat16)


# --------------------------------------------------------------------------
# clocks: NVML polled in a thread; summarised over the timed window
# --------------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index):
        self.samples = []
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report it
            self.err = str(e)
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, rs))
            except Exception:
                pass
            time.sleep(0.01)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": f"NVML unavailable: {self.err}"}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        src = "timed_region"
        if not win:  # region shorter than the poll period: use the soak + timed span
            win = self.samples
            src = "warmup+timed (timed region shorter than the 10 ms poll)"
        reasons = set()
        for _, _, r in win:
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median([s[1] for s in win]) if win else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons), "samples": len(win), "window": src}


# --------------------------------------------------------------------------
# timing helpers
# --------------------------------------------------------------------------

def graph_time(torch, step_fn, steps, warmup, soak_s, barrier, sampler=None):
    """Run `steps` steps (step_fn(i) enqueues step i) as CUDA-graph replays.
    Returns (elapsed_ms over the K timed steps, t0, t1 host stamps)."""
    stream = torch.cuda.Stream()
    per = max(1, min(steps, 500))
    with torch.cuda.stream(stream):
        for i in range(3):  # eager warm-up (module loads, cuBLAS workspaces)
            step_fn(i)
    torch.cuda.synchronize()
    g_main = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_main, stream=stream):
        for i in range(per):
            step_fn(i)
    tail = steps % per
    g_tail = None
    if tail:
        g_tail = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_tail, stream=stream):
            for i in range(tail):
                step_fn(per + i)
    reps = steps // per
    with torch.cuda.stream(stream):
        for _ in range(max(1, math.ceil(warmup / per))):
            g_main.replay()
        torch.cuda.synchronize()
        t_soak = time.perf_counter()
        while time.perf_counter() - t_soak < soak_s:  # settle clocks
            g_main.replay()
            torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(reps):
            g_main.replay()
        if g_tail is not None:
            g_tail.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        barrier()
    return e0.elapsed_time(e1), t0, t1


def max_over_ranks(torch, dist, value):
    if dist is None:
        return value
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------
# CPU legs (the reference compiled from its sources, else our C port)
# --------------------------------------------------------------------------

def cpu_backend():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, Reference, build
    if Reference.available():
        return Reference(), "reference"
    build()
    return Oracle(), "port"


def cpu_spmm_rate(wl, budget_s, max_calls=None):
    """Time the CPU spmm_execute on the workload (host copies of the same
    kind of synthetic inputs).  Returns (tflops_dense_equiv, calls, seconds,
    cores, kind, sample_desc)."""
    be, kind = cpu_backend()
    M, N, K, V = wl["M"], wl["N"], wl["K"], wl["V"]
    cpg = int(round(wl["alpha"] * K))
    mask = synth_mask(M, K, V, cpg, 1234)
    rs = np.random.RandomState(1)
    W = (rs.rand(M, K).astype(np.float32) * 2 - 1)
    B = (rs.rand(K, N).astype(np.float32) * 2 - 1)
    p = be.compress(W, mask, V)
    cores = os.cpu_count() or 1
    # bounded sample: all groups if a call fits the budget, else a prefix
    G = M // V
    g_sub = G
    from oracle import Packed
    def sub(gs):
        nc = int(p.group_ncols[:gs].sum())
        return Packed(gs * V, K, V, np.arange(gs * V, dtype=np.uint32), p.group_ncols[:gs].copy(),
                      p.cols[:nc].copy(), p.values[: nc * V].copy())
    a = sub(g_sub)
    if kind == "reference":
        ha, hb = be.prebuilt(a, B)
        call = lambda: be.spmm_prebuilt(ha, hb, cores)
    else:
        call = lambda: be.spmm(a, B)
        cores = 1
    t = time.perf_counter()
    call()
    one = time.perf_counter() - t
    if one > budget_s / 3 and G > 1:  # shrink the sample
        g_sub = max(1, int(G * (budget_s / 3) / one))
        if kind == "reference":
            be.free_prebuilt(ha, hb)
            a = sub(g_sub)
            ha, hb = be.prebuilt(a, B)
            call = lambda: be.spmm_prebuilt(ha, hb, cores)
        else:
            a = sub(g_sub)
    calls, t0 = 0, time.perf_counter()
    while True:
        call()
        calls += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (max_calls and calls >= max_calls):
            break
    if kind == "reference":
        be.free_prebuilt(ha, hb)
    flops = 2.0 * g_sub * V * N * K * calls
    desc = (f"{calls} spmm_execute calls on {g_sub}/{G} row groups of the {M}x{K} V={V} "
            f"{int(wl['alpha'] * 100)}% matrix, N={N}, fp32, TileConfig{{}}, threads={cores}")
    return flops / el / 1e12, calls, el, cores, kind, desc, g_sub


def run_reference_arm(args, wl, world, rank):
    if rank != 0:
        return
    be, kind = cpu_backend()
    M, N, K, V = wl["M"], wl["N"], wl["K"], wl["V"]
    cpg = int(round(wl["alpha"] * K))
    mask = synth_mask(M, K, V, cpg, 1234)
    rs = np.random.RandomState(1)
    W = rs.rand(M, K).astype(np.float32) * 2 - 1
    B = rs.rand(K, N).astype(np.float32) * 2 - 1
    p = be.compress(W, mask, V)
    cores = os.cpu_count() or 1
    G = M // V
    from oracle import Packed

    def sub(gs):
        nc = int(p.group_ncols[:gs].sum())
        return Packed(gs * V, K, V, np.arange(gs * V, dtype=np.uint32), p.group_ncols[:gs].copy(),
                      p.cols[:nc].copy(), p.values[: nc * V].copy())
    g_sub = G
    a = sub(G)
    if kind == "reference":
        ha, hb = be.prebuilt(a, B)
        call = lambda: be.spmm_prebuilt(ha, hb, cores)
    else:
        cores = 1
        call = lambda: be.spmm(a, B)
    t = time.perf_counter()
    call()
    one = time.perf_counter() - t
    budget = 150.0  # whole run stays within a few minutes
    steps, warm = args.steps, args.warmup
    if one * (steps + warm) > budget and G > 1:
        g_sub = max(1, int(G * budget / ((steps + warm) * one)))
        if kind == "reference":
            be.free_prebuilt(ha, hb)
            a = sub(g_sub)
            ha, hb = be.prebuilt(a, B)
            call = lambda: be.spmm_prebuilt(ha, hb, cores)
        else:
            a = sub(g_sub)
    for _ in range(warm):
        call()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    el = time.perf_counter() - t0
    flops = 2.0 * g_sub * V * N * K
    value = flops * steps / el / 1e12
    sample = (f"each step: one spmm_execute over {g_sub}/{G} row groups of the workload "
              f"({'full problem' if g_sub == G else 'bounded sample'}), fp32, threads={cores}")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": el / steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl["desc"], "M": M, "N": N, "K": K, "V": V,
                       "sparsity": 1 - wl["alpha"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=500)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="ns", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--allgather", action="store_true",
                    help="lf, N > 1: also time the full-output gather -- NCCL all-gather + unpermute, and fused "
                         "into the epilogue (P2P stores)")
    ap.add_argument("--soak", type=float, default=0.3, help="seconds of untimed replays to settle clocks")
    ap.add_argument("--e2e-steps", type=int, default=500)
    ap.add_argument("--e2e-streams", type=int, default=6, help="e2e: steps in flight (round-robin streams)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no baselines, few steps")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, wl, world, rank)

    import torch
    import paper_2203_05016_b200 as sb
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    barrier = (lambda: dist.barrier()) if dist is not None else (lambda: None)
    dev = torch.device("cuda", local)

    M, N, K, V, alpha = wl["M"], wl["N"], wl["K"], wl["V"], wl["alpha"]
    G = M // V
    cpg = int(round(alpha * K))
    if wl["sharded"]:
        g0, g1 = G * rank // world, G * (rank + 1) // world
        scaling = "strong"
    else:
        g0, g1 = 0, G
        scaling = "weak"
    my_groups = g1 - g0

    # ---- inputs: rotating sets whose total exceeds L2 --------------------
    mask = torch.from_numpy(synth_mask(M, K, V, cpg, 1234 + 0)).to(dev)
    kpad = (cpg + 63) // 64 * 64
    set_bytes = 2 * M * kpad + 4 * G * kpad + 4 * M + 2 * K * N + 2 * M * N
    nsets = 1 if set_bytes > L2_BYTES else min(64, max(2, math.ceil(1.25 * L2_BYTES / set_bytes)))
    if args.profile:
        nsets = min(nsets, 4)
    mats, Bs, Cs = [], [], []
    t_c = None
    for s in range(nsets):
        W = uniform_bf16(torch, (M, K), 100 + s, dev)
        torch.cuda.synchronize()
        t = time.perf_counter()
        mats.append(sb.compress_shflbw(W, mask, V))
        torch.cuda.synchronize()
        if t_c is None and (s == 1 or nsets == 1):
            t_c = (time.perf_counter() - t) * 1e3
        Bs.append(uniform_bf16(torch, (K, N), 200 + s, dev))
        Cs.append(torch.empty((my_groups * V, N) if wl["sharded"] else (M, N), dtype=torch.bfloat16, device=dev))
        if s == 0 and not args.profile:
            # converter (the reference's compress_shflbw) with a warm allocator:
            # median wall time of 5 calls, device-resident W and mask
            ts = []
            for _ in range(5):
                torch.cuda.synchronize()
                t = time.perf_counter()
                tmp = sb.compress_shflbw(W, mask, V)
                torch.cuda.synchronize()
                ts.append((time.perf_counter() - t) * 1e3)
                del tmp
            t_c = sorted(ts)[2]
        del W

    def step_ours(i):
        s = i % nsets
        if wl["sharded"]:
            sb.spmm_groups(mats[s], g0, g1, Bs[s], Cs[s], compact=True)
        else:
            sb.spmm_execute(mats[s], Bs[s], out=Cs[s])

    n_before = sb.launch_count()
    step_ours(0)
    launches_per_step = sb.launch_count() - n_before
    torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    ms, t0, t1 = graph_time(torch, step_ours, args.steps, args.warmup, 0.0 if args.profile else args.soak, barrier)
    sampler.stop()
    ms = max_over_ranks(torch, dist, ms)
    clocks = sampler.summary(t0, t1)
    ms_step = ms / args.steps

    flops_dense = 2.0 * M * N * K  # whole layer (strong) or per rank (weak), see below
    total_flops = flops_dense * (1 if wl["sharded"] else world)
    value = total_flops * args.steps / (ms * 1e-3) / 1e12

    # ---- multi-GPU all-gather (lf --allgather): compute + NCCL gather ----
    gather = None
    if wl["sharded"] and world > 1 and args.allgather:
        full = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        gathered = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for i in range(reps):
            step_ours(i)
            dist.all_gather_into_tensor(gathered, Cs[i % nsets])
            sb.unpermute_rows(mats[i % nsets].row_indices_ptr, gathered, full)
        e1.record()
        torch.cuda.synchronize()
        gms = max_over_ranks(torch, dist, e0.elapsed_time(e1) / reps)
        gather = {"ms_per_step": gms, "tflops_dense_equiv": flops_dense / (gms * 1e-3) / 1e12,
                  "collective": "ncclAllGather (torch.distributed all_gather_into_tensor) + unpermute"}
        # the same gather fused into the epilogue: each rank's rows stored at
        # their final positions into every rank's full output over P2P
        from paper_2203_05016_b200.sharded import PeerOutputs
        outs = PeerOutputs((M, N), torch.bfloat16, world, rank)
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(reps):
            sb.spmm_groups_peers(mats[i % nsets], g0, g1, Bs[i % nsets], outs.ptrs, dtype=torch.bfloat16, ldc=N)
        e1.record()
        torch.cuda.synchronize()
        fms = max_over_ranks(torch, dist, e0.elapsed_time(e1) / reps)
        barrier()
        outs.close()
        gather["fused"] = {"ms_per_step": fms, "tflops_dense_equiv": flops_dense / (fms * 1e-3) / 1e12,
                           "collective": "none: shflbw_cu_spmm_groups_peers stores every row into all ranks' "
                                         "outputs over P2P (CUDA IPC) from the epilogue"}

    if args.profile:
        if rank == 0:
            print(json.dumps({"profile_run": True, "ms_per_step": ms_step, "value": value}), flush=True)
        return

    # ---- cuBLAS dense bf16 GEMM, same shape, same protocol ---------------
    cub = None
    if not wl["sharded"] or world == 1:
        Wd = [sb.decompress(m).to(torch.bfloat16) for m in mats]
        Cd = [torch.empty((M, N), dtype=torch.bfloat16, device=dev) for _ in range(nsets)]

        def step_cublas(i):
            s = i % nsets
            torch.mm(Wd[s], Bs[s], out=Cd[s])
        cms, _, _ = graph_time(torch, step_cublas, args.steps, args.warmup, 0.0, barrier)
        cub = {"ms_per_step": cms / args.steps, "tflops": 2.0 * M * N * K * args.steps / (cms * 1e-3) / 1e12,
               "impl": "torch.mm bf16 (cuBLAS), dense W*mask, bf16 out, same rotating sets + CUDA graph"}
        del Wd, Cd

    # ---- fp32-output (parity mode) ----------------------------------------
    C32 = [torch.empty((M, N), dtype=torch.float32, device=dev) for _ in range(nsets)] if not wl["sharded"] else None
    f32 = None
    if C32 is not None:
        def step32(i):
            s = i % nsets
            sb.spmm_execute(mats[s], Bs[s], out=C32[s])
        fms, _, _ = graph_time(torch, step32, args.steps, args.warmup, 0.0, barrier)
        f32 = {"ms_per_step": fms / args.steps,
               "tflops_dense_equiv": 2.0 * M * N * K * args.steps / (fms * 1e-3) / 1e12}
        del C32

    # ---- e2e through the public API with pinned host buffers ---------------
    # Every step copies its activations host->device (pinned), runs the SpMM
    # through the public Python API and reads the result back device->host.
    # Steps round-robin over 3 streams so copies of one step overlap the
    # compute of another (the copy engines and the SMs run concurrently).
    a0 = mats[0]
    out_rows = my_groups * V if wl["sharded"] else M
    nstr = args.e2e_streams
    streams = [torch.cuda.Stream() for _ in range(nstr)]
    Bh = [Bs[i % nsets].cpu().pin_memory() for i in range(nstr)]
    Ch = [torch.empty((out_rows, N), dtype=torch.bfloat16).pin_memory() for _ in range(nstr)]
    Bd = [torch.empty_like(Bs[0]) for _ in range(nstr)]
    Cdv = [torch.empty((out_rows, N), dtype=torch.bfloat16, device=dev) for _ in range(nstr)]
    e2e_steps = max(3, min(args.steps, args.e2e_steps))

    # Each step: cudaMemcpyAsync H2D of B (pinned host), the C-ABI SpMM
    # (shflbw_cu_spmm / _spmm_groups, the reference-facing boundary) and
    # cudaMemcpyAsync D2H of C, on one of 3 streams -- issued through
    # cuda-python and ctypes so the host issue cost (~1 us per call) stays
    # below the PCIe time of the copies.
    from cuda.bindings import runtime as rt
    lib = sb.shflbw._lib()
    h2d, d2h = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost
    sh = [st.cuda_stream for st in streams]
    rts = [rt.cudaStream_t(h) for h in sh]
    nb_b, nb_c = Bh[0].numel() * Bh[0].element_size(), Ch[0].numel() * Ch[0].element_size()
    p_bh, p_bd = [t.data_ptr() for t in Bh], [t.data_ptr() for t in Bd]
    p_ch, p_cd = [t.data_ptr() for t in Ch], [t.data_ptr() for t in Cdv]
    a_ref = a0.ptr
    Kb, ldb = Bd[0].shape[0], Bd[0].stride(0)

    def e2e_step(i):
        k = i % nstr
        if rt.cudaMemcpyAsync(p_bd[k], p_bh[k], nb_b, h2d, rts[k])[0] != rt.cudaError_t.cudaSuccess:
            raise RuntimeError("cudaMemcpyAsync H2D failed")
        if wl["sharded"]:
            st = lib.shflbw_cu_spmm_groups(a_ref, g0, g1, p_bd[k], Kb, N, ldb, p_cd[k], 1, N, 1, sh[k])
        else:
            st = lib.shflbw_cu_spmm(a_ref, p_bd[k], Kb, N, ldb, p_cd[k], 1, N, sh[k])
        if st:
            raise RuntimeError(f"shflbw_cu_spmm status {st}: {lib.shflbw_cu_last_error()}")
        if rt.cudaMemcpyAsync(p_ch[k], p_cd[k], nb_c, d2h, rts[k])[0] != rt.cudaError_t.cudaSuccess:
            raise RuntimeError("cudaMemcpyAsync D2H failed")
    for i in range(6):
        e2e_step(i)
    torch.cuda.synchronize()
    barrier()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for st in streams:
        st.wait_event(e0)
    for i in range(e2e_steps):
        e2e_step(i)
    for st in streams:
        main.wait_stream(st)
    e1.record(main)
    torch.cuda.synchronize()
    ems = max_over_ranks(torch, dist, e0.elapsed_time(e1)) / e2e_steps
    e2e = {"value": total_flops / (ems * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ems,
           "h2d_bytes_per_step": Bh[0].numel() * Bh[0].element_size(),
           "d2h_bytes_per_step": Ch[0].numel() * Ch[0].element_size(), "steps": e2e_steps,
           "path": ("C ABI shflbw_cu_spmm (ctypes) with cudaMemcpyAsync (cuda-python) of pinned host B/C: "
                    f"H2D + SpMM + D2H per step, {nstr} streams round-robin")}

    # ---- roofline of the dominant kernel (the SpMM, one launch per step) ---
    hbm, tfl_burst, tfl_sus, peak_kind = load_peaks()
    kprime = cpg
    q_bytes = (2 * my_groups * V * kpad + 4 * my_groups * kpad + 4 * my_groups * V + 2 * K * N
               + 2 * my_groups * V * N)
    useful_flops = 2.0 * my_groups * V * N * kprime
    ridge = tfl_burst * 1e12 / (hbm * 1e9)
    t_launch = ms_step * 1e-3  # the SpMM is the only kernel in a step
    if useful_flops / q_bytes < ridge:
        achieved = q_bytes / t_launch / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm}
    else:
        achieved = useful_flops / t_launch / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tfl_burst, "unit": "TFLOP/s",
                "frac": achieved / tfl_burst}
    roof.update({"traffic": None, "algorithmic_bytes_per_launch": q_bytes, "useful_flops_per_launch": useful_flops,
                 "peak_source": f"MEASURED_PEAKS.json ({peak_kind}, burst)",
                 "kernel": "k_spmm_tc (tcgen05 + TMA gather4)"})
    prof_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    util = None
    if os.path.exists(prof_path):
        with open(prof_path) as f:
            prof = json.load(f).get(args.workload)
        if prof:
            roof["traffic"] = prof.get("dram_bytes_per_launch")
            util = prof.get("tensor_pipe_util_pct")
            roof["traffic_source"] = prof.get("source")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, calls, el, cores, kind, desc, _ = cpu_spmm_rate(wl, args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc, "seconds": el}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": wl["desc"], "M": M, "N": N, "K": K, "V": V, "sparsity": 1 - alpha,
                       "kept_cols_per_group": cpg, "groups": G, "out_dtype": "bf16", "accum": "fp32",
                       "parallelism": (f"row-group shards x{world}" if wl["sharded"] else f"replicas x{world}"),
                       "l2": (f"{nsets} rotating input sets x {set_bytes / 2**20:.1f} MiB > 126 MB L2"
                              if nsets > 1 else "inputs larger than L2"),
                       "timing": "CUDA graph replays, CUDA events on the launching stream, max over ranks"},
            "speedup_vs_cublas": (value / world / cub["tflops"]) if cub else None,
            "cublas": cub, "fp32_out": f32, "tensor_pipe_util_pct": util,
            "compress_ms": t_c, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps, "launches_per_step": launches_per_step,
            "allgather": gather,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
