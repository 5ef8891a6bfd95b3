"""Short timing of a fixed case list (development, for scripts/ab.sh)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch  # noqa: E402

import paper_2203_05016_b200 as sb  # noqa: E402
import sweep  # noqa: E402

dev = torch.device("cuda", 0)
for kv in [x for x in os.environ.get("SBW_OPTS", "").split(",") if x]:  # e.g. SBW_OPTS=gather_warps=8
    k, v = kv.split("=")
    sb.set_option(k, int(v))
only = sys.argv[1].split(",") if len(sys.argv) > 1 else ["ns", "ffn2", "gnmt90", "conv56", "conv14"]
cases = {
    "ns": lambda: sweep.spmm_row("ns", 2048, 128, 2048, 64, 0.25, 2000, dev),
    "ffn2": lambda: sweep.spmm_row("ffn2", 512, 4096, 2048, 64, 0.25, 1000, dev),
    "ffn1": lambda: sweep.spmm_row("ffn1", 2048, 4096, 512, 64, 0.25, 1000, dev),
    "ffn1_50": lambda: sweep.spmm_row("ffn1_50", 2048, 4096, 512, 64, 0.5, 1000, dev),
    "ffn2_v32": lambda: sweep.spmm_row("ffn2_v32", 512, 4096, 2048, 32, 0.25, 1000, dev),
    "ns_v32": lambda: sweep.spmm_row("ns_v32", 2048, 128, 2048, 32, 0.25, 2000, dev),
    "ns_v128": lambda: sweep.spmm_row("ns_v128", 2048, 128, 2048, 128, 0.25, 2000, dev),
    "gnmt50": lambda: sweep.spmm_row("gnmt50", 4096, 128, 1024, 64, 0.5, 2000, dev),
    "gnmt75": lambda: sweep.spmm_row("gnmt75", 4096, 128, 1024, 64, 0.25, 2000, dev),
    "attn128": lambda: sweep.spmm_row("attn128", 512, 128, 512, 64, 0.25, 2000, dev),
    "ffn1_128": lambda: sweep.spmm_row("ffn1_128", 2048, 128, 512, 64, 0.25, 2000, dev),
    "ffn2_128": lambda: sweep.spmm_row("ffn2_128", 512, 128, 2048, 64, 0.25, 2000, dev),
    "gnmt95": lambda: sweep.spmm_row("gnmt95", 4096, 128, 1024, 64, 0.05, 2000, dev),
    "gnmt90": lambda: sweep.spmm_row("gnmt90", 4096, 128, 1024, 64, 0.1, 2000, dev),
    "lf": lambda: sweep.spmm_row("lf", 16384, 8192, 4096, 64, 0.25, 20, dev),
    "conv56": lambda: sweep.conv_row("conv56", 64, 56, 64, 3, 1, 32, 64, 0.25, 300, dev),
    "conv28": lambda: sweep.conv_row("conv28", 128, 28, 128, 3, 1, 32, 64, 0.25, 300, dev),
    "conv14": lambda: sweep.conv_row("conv14", 256, 14, 256, 3, 1, 32, 64, 0.25, 300, dev),
    "conv7": lambda: sweep.conv_row("conv7", 512, 7, 512, 3, 1, 32, 64, 0.25, 300, dev),
    "c1x1_56": lambda: sweep.conv_row("c1x1_56", 256, 56, 64, 1, 0, 32, 64, 0.25, 300, dev),
    "c1x1_14": lambda: sweep.conv_row("c1x1_14", 1024, 14, 256, 1, 0, 32, 64, 0.25, 300, dev),
    "attn4096": lambda: sweep.spmm_row("attn4096", 512, 4096, 512, 64, 0.25, 1000, dev),
    "ffn1_90": lambda: sweep.spmm_row("ffn1_90", 2048, 4096, 512, 64, 0.1, 1000, dev),
    "ffn2_v128": lambda: sweep.spmm_row("ffn2_v128", 512, 4096, 2048, 128, 0.25, 1000, dev),
}
out = {}
for k in only:
    if k.startswith("c_"):  # ad-hoc 1x1 conv, batch 32, 75 %: c_Cin_H_Cout
        C_, H_, F_ = (int(x) for x in k[2:].split("_"))
        r = sweep.conv_row(k, C_, H_, F_, 1, 0, 32, 64, 0.25, 300, dev)
        out[k] = (round(r["us"], 2), round(r["dense_us"], 2))
        continue
    if k.startswith("s_"):  # ad-hoc SpMM: s_M_N_K_V_alpha
        M_, N_, K_, V_, a_ = k[2:].split("_")
        r = sweep.spmm_row(k, int(M_), int(N_), int(K_), int(V_), float(a_), 1000, dev)
        out[k] = (round(r["us"], 2), round(r["dense_us"], 2))
        continue
    r = cases[k]()
    out[k] = (round(r["us"], 2), round(r["dense_us"], 2))
print(json.dumps(out))
