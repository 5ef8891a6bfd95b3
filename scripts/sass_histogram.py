"""SASS instruction histogram of the tcgen05 kernels in the built library
(evidence that the hot path is tcgen05 + TMA: UTCHMMA, UTMALDG.*GATHER4,
LDTM, STSM), written to profiles/sass_<tag>.md.

    python scripts/sass_histogram.py <tag>
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2203_05016_b200", "lib", "libshflbw_b200.so")
KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG.2D.GATHER4", "UTMALDG.2D.GATHER4.MULTICAST", "UTMALDG.2D", "UBLKCP",
        "LDTM", "STSM", "STAS", "SYNCS.ARRIVE", "SYNCS.PHASECHK", "ELECT", "R2UR.BROADCAST", "LDGSTS", "HMMA"]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r2"
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
        if m:
            op = m.group(1)
            c = funcs[cur]
            c["total"] += 1
            for k in KEYS:
                if op == k or op.startswith(k + "."):
                    c[k] += 1
    sel = {f: c for f, c in funcs.items() if "k_spmm_tc" in f or "k_spmm_persist" in f}
    tot = collections.Counter()
    for c in sel.values():
        tot.update(c)
    lines = [f"# SASS histogram ({tag}): tcgen05 kernels in libshflbw_b200.so", "",
             f"{len(sel)} instantiations of k_spmm_tc / k_spmm_persist (cuobjdump -sass).", "",
             "| opcode | count (all instantiations) |", "|---|---|"]
    for k in ["total"] + KEYS:
        lines.append(f"| {k} | {tot[k]} |")
    lines += ["", "North-star kernel (`k_spmm_tc<BF16, VS=32, CS=4, KIND=0, 2x2, GW=4>`):", "",
              "| opcode | count |", "|---|---|"]
    ns = [c for f, c in sel.items() if f.startswith("_ZN3sbw2tc9k_spmm_tcILi1ELi32ELi4ELi0ELi2ELi4E")]
    if ns:
        for k in ["total"] + KEYS:
            lines.append(f"| {k} | {ns[0][k]} |")
    path = os.path.join(ROOT, "profiles", f"sass_{tag}.md")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
