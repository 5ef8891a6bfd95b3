"""BASELINE.json configuration sweep on one GPU (not the driver's bench line).

    python scripts/sweep.py [--steps 300] [--out profiles/sweep_r1]

For every configuration of BASELINE.json (north-star variants, Transformer-
base linear layers, GNMT gate GEMMs over a sparsity sweep, ResNet-50
stride-1 convs at batch 32, the large FFN on one GPU) it times the Shfl-BW
kernel and the dense library baseline (cuBLAS bf16 GEMM via torch.mm /
cuDNN conv via torch.nn.functional.conv2d) with the bench protocol
(rotating input sets > L2, CUDA graphs, CUDA events) and writes a markdown
table + JSON.  Dense-equivalent TFLOP/s = dense FLOPs / time.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_05016_b200 as sb  # noqa: E402

SPMM = [  # name, M, N, K, V, alpha
    ("north star V=64", 2048, 128, 2048, 64, 0.25),
    ("north star V=32", 2048, 128, 2048, 32, 0.25),
    ("north star V=128", 2048, 128, 2048, 128, 0.25),
    ("attn proj 512x512 N=128", 512, 128, 512, 64, 0.25),
    ("FFN1 2048x512 N=128", 2048, 128, 512, 64, 0.25),
    ("FFN2 512x2048 N=128", 512, 128, 2048, 64, 0.25),
    ("attn proj 512x512 N=4096", 512, 4096, 512, 64, 0.25),
    ("FFN1 2048x512 N=4096 50%", 2048, 4096, 512, 64, 0.5),
    ("FFN1 2048x512 N=4096 75%", 2048, 4096, 512, 64, 0.25),
    ("FFN1 2048x512 N=4096 90%", 2048, 4096, 512, 64, 0.1),
    ("FFN2 512x2048 N=4096 75%", 512, 4096, 2048, 64, 0.25),
    ("FFN2 512x2048 N=4096 V=32", 512, 4096, 2048, 32, 0.25),
    ("FFN2 512x2048 N=4096 V=128", 512, 4096, 2048, 128, 0.25),
    ("GNMT 4096x1024 N=128 50%", 4096, 128, 1024, 64, 0.5),
    ("GNMT 4096x1024 N=128 75%", 4096, 128, 1024, 64, 0.25),
    ("GNMT 4096x1024 N=128 90%", 4096, 128, 1024, 64, 0.1),
    ("GNMT 4096x1024 N=128 95%", 4096, 128, 1024, 64, 0.05),
    ("large FFN 16384x4096 N=8192", 16384, 8192, 4096, 64, 0.25),
]
CONV = [  # name, C, H, Kf, R, pad, Nb, V, alpha
    ("ResNet 3x3 64->64 @56", 64, 56, 64, 3, 1, 32, 64, 0.25),
    ("ResNet 3x3 128->128 @28", 128, 28, 128, 3, 1, 32, 64, 0.25),
    ("ResNet 3x3 256->256 @14", 256, 14, 256, 3, 1, 32, 64, 0.25),
    ("ResNet 3x3 512->512 @7", 512, 7, 512, 3, 1, 32, 64, 0.25),
    ("ResNet 1x1 256->64 @56", 256, 56, 64, 1, 0, 32, 64, 0.25),
    ("ResNet 1x1 1024->256 @14", 1024, 14, 256, 1, 0, 32, 64, 0.25),
]


def nsets_for(bytes_per_set):
    return 1 if bytes_per_set > bench.L2_BYTES else min(64, max(2, math.ceil(1.25 * bench.L2_BYTES / bytes_per_set)))


def time_steps(step, steps):
    ms, _, _ = bench.graph_time(torch, step, steps, 20, 0.05, lambda: None)
    return ms / steps


def spmm_row(name, M, N, K, V, alpha, steps, dev):
    cpg = int(round(alpha * K))
    kpad = (cpg + 63) // 64 * 64
    # enough rotating sets that EACH implementation's own operands exceed L2
    # (ours: packed weights + indices + B + C; dense: W + B + C)
    n = max(nsets_for(2 * M * kpad + 4 * (M // V) * kpad + 2 * K * N + 2 * M * N),
            nsets_for(2 * M * K + 2 * K * N + 2 * M * N))
    if os.environ.get("SBW_WARM"):  # development: one L2-resident operand set
        n = 1
    mask = torch.from_numpy(bench.synth_mask(M, K, V, cpg, 1234)).to(dev)
    mats, Wd, Bs, Cs, Cd = [], [], [], [], []
    for s in range(n):
        W = bench.uniform16(torch, (M, K), 100 + s, dev)
        mats.append(sb.compress_shflbw(W, mask, V))
        Wd.append((W * mask).contiguous())
        Bs.append(bench.uniform16(torch, (K, N), 200 + s, dev))
        Cs.append(torch.empty((M, N), dtype=torch.bfloat16, device=dev))
        Cd.append(torch.empty((M, N), dtype=torch.bfloat16, device=dev))
    t_ours = time_steps(lambda i: sb.spmm_execute(mats[i % n], Bs[i % n], out=Cs[i % n]), steps)
    plan = sb.last_plan()
    t_dense = time_steps(lambda i: torch.mm(Wd[i % n], Bs[i % n], out=Cd[i % n]), steps)
    err = (Cs[0].float() - Cd[0].float()).norm() / Cd[0].float().norm()
    flops = 2.0 * M * N * K
    q = 2 * M * kpad + 4 * (M // V) * kpad + 4 * M + 2 * K * N + 2 * M * N
    return {"name": name, "M": M, "N": N, "K": K, "V": V, "sparsity": 1 - alpha, "us": t_ours * 1e3,
            "dense_us": t_dense * 1e3, "tflops_dense_equiv": flops / (t_ours * 1e-3) / 1e12,
            "dense_tflops": flops / (t_dense * 1e-3) / 1e12, "speedup": t_dense / t_ours,
            "hbm_gbs": q / (t_ours * 1e-3) / 1e9, "useful_tflops": flops * alpha / (t_ours * 1e-3) / 1e12,
            "rel_err_vs_dense_bf16": float(err), "sets": n, "plan": plan}


def conv_row(name, C, H, Kf, R, pad, Nb, V, alpha, steps, dev):
    crs = C * R * R
    cpg = int(round(alpha * crs))
    n = max(nsets_for(2 * C * H * H * Nb * 2 + 2 * Kf * crs // 4), nsets_for(2 * C * H * H * Nb * 2 + 2 * Kf * crs))
    mask = torch.from_numpy(bench.synth_mask(Kf, crs, V, cpg, 1234)).to(dev)
    geo = sb.ConvGeometry(R, R, 1, pad)
    P = H + 2 * pad - R + 1
    mats, xs, outs, Wc, xc = [], [], [], [], []
    for s in range(n):
        W = bench.uniform16(torch, (Kf, crs), 100 + s, dev)
        mats.append(sb.conv_prepare(sb.compress_shflbw(W, mask, V), geo))  # one-time conv weight order
        Wc.append((W * mask).reshape(Kf, C, R, R).contiguous())
        x = bench.uniform16(torch, (C, H, H, Nb), 300 + s, dev)
        xs.append(x)
        xc.append(x.permute(3, 0, 1, 2).contiguous(memory_format=torch.channels_last))  # NCHW, channels-last
        outs.append(torch.empty((Kf, P, P, Nb), dtype=torch.bfloat16, device=dev))
    lib = sb.shflbw._lib()

    def step_ours(i):
        k = i % n
        st = lib.shflbw_cu_conv2d(mats[k].ptr, xs[k].data_ptr(), C, H, H, Nb, R, R, 1, pad, outs[k].data_ptr(),
                                  1, torch.cuda.current_stream().cuda_stream)
        assert st == 0
    t_ours = time_steps(step_ours, steps)
    plan = sb.last_plan()
    Wcl = [w.contiguous(memory_format=torch.channels_last) for w in Wc]
    t_dense = time_steps(lambda i: torch.nn.functional.conv2d(xc[i % n], Wcl[i % n], padding=pad), steps)
    ref = torch.nn.functional.conv2d(xc[0], Wcl[0], padding=pad).float().permute(1, 2, 3, 0)
    err = (outs[0].float() - ref).norm() / ref.norm()
    flops = 2.0 * Kf * crs * P * P * Nb
    return {"name": name, "C": C, "H": H, "Kf": Kf, "R": R, "Nb": Nb, "V": V, "sparsity": 1 - alpha,
            "us": t_ours * 1e3, "dense_us": t_dense * 1e3, "tflops_dense_equiv": flops / (t_ours * 1e-3) / 1e12,
            "dense_tflops": flops / (t_dense * 1e-3) / 1e12, "speedup": t_dense / t_ours,
            "rel_err_vs_cudnn_bf16": float(err), "sets": n, "plan": plan}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep"))
    ap.add_argument("--only", default="")
    ap.add_argument("--grid", default="", help="'transformer': BASELINE configs[1] in full -- (M, K) in "
                    "{512x512, 2048x512, 512x2048} x N in {128, 512, 1024, 4096} x 50/75/90 % x V in {32, 64, 128}")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rows = []
    spmm_cfgs, conv_cfgs = SPMM, CONV
    if args.grid == "resnet":  # every stride-1 ResNet-50 bottleneck conv, batch 32, 75 %
        spmm_cfgs = []
        conv_cfgs = []
        for stage, (Cin, mid, Cout, H) in enumerate(((256, 64, 256, 56), (512, 128, 512, 28),
                                                      (1024, 256, 1024, 14), (2048, 512, 2048, 7))):
            conv_cfgs += [(f"ResNet 1x1 {Cin}->{mid} @{H}", Cin, H, mid, 1, 0, 32, 64, 0.25),
                          (f"ResNet 3x3 {mid}->{mid} @{H}", mid, H, mid, 3, 1, 32, 64, 0.25),
                          (f"ResNet 1x1 {mid}->{Cout} @{H}", mid, H, Cout, 1, 0, 32, 64, 0.25)]
        conv_cfgs.insert(0, ("ResNet 1x1 64->64 @56", 64, 56, 64, 1, 0, 32, 64, 0.25))
    if args.grid == "transformer":
        spmm_cfgs, conv_cfgs = [], []
        for nm, M, K in (("attn proj", 512, 512), ("FFN1", 2048, 512), ("FFN2", 512, 2048)):
            for N in (128, 512, 1024, 4096):
                for alpha in (0.5, 0.25, 0.1):
                    for V in (32, 64, 128):
                        spmm_cfgs.append((f"{nm} {M}x{K} N={N} {round((1 - alpha) * 100)}% V={V}", M, N, K, V, alpha))
    for cfg in spmm_cfgs:
        if args.only and args.only not in cfg[0]:
            continue
        rows.append(spmm_row(*cfg, args.steps if cfg[1] * cfg[2] < 1 << 26 else 20, dev))
        print(json.dumps(rows[-1]), flush=True)
    for cfg in conv_cfgs:
        if args.only and args.only not in cfg[0]:
            continue
        rows.append(conv_row(*cfg, args.steps, dev))
        print(json.dumps(rows[-1]), flush=True)
    lines = ["| config | Shfl-BW us | dense us (cuBLAS/cuDNN) | dense-eq TFLOP/s | speed-up | rel err vs dense | plan |",
             "|---|---|---|---|---|---|---|"]
    for r in rows:
        e = r.get("rel_err_vs_dense_bf16", r.get("rel_err_vs_cudnn_bf16"))
        lines.append(f"| {r['name']} | {r['us']:.2f} | {r['dense_us']:.2f} | {r['tflops_dense_equiv']:.0f} | "
                     f"{r['speedup']:.2f}x | {e:.1e} | {r.get('plan', '')} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(args.out + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
