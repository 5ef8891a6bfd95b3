#!/bin/bash
# Development: every listed option setting over the BASELINE SpMM / conv cases
# (scripts/ab_cases.py), one JSON line per setting.
cd $GRAFT_REPO_ROOT
C=ns,ns_v32,ns_v128,attn128,ffn1_128,ffn2_128,attn4096,ffn1,ffn1_50,ffn1_90,ffn2,ffn2_v32,ffn2_v128,gnmt50,gnmt75,gnmt90,gnmt95,conv56,conv28,conv14,conv7,c1x1_56,c1x1_14
for o in split=0 gather_warps=4 gather_warps=8 stages=2 stages=3 stages=4 stages=6 tile_n=64 tile_n=128 pdl_trigger=1 pdl_trigger=-1 prefetch=16 prefetch=-1 split=0; do
  echo "== $o"
  SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C 2>&1 | grep '^{'
done
