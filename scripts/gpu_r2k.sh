#!/bin/bash
cd $GRAFT_REPO_ROOT
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95,attn128,ffn1_128,ffn2_128,ffn2,ffn1,ffn2_v32
for o in "gather_issue=0" "gather_issue=1" "gather_issue=0,gather_warps=8" "gather_issue=1,gather_warps=8" "gather_issue=0,tile_n=64" "gather_issue=1,tile_n=64" "gather_issue=0,tile_n=64,gather_warps=8" "gather_issue=1,tile_n=64,gather_warps=8" "gather_issue=0,tile_n=128"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
done
