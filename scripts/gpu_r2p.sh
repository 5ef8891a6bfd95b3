#!/bin/bash
cd $GRAFT_REPO_ROOT
for o in "split=0" "tile_n=64,split=4,split_mode=2" "gather_warps=8" "tile_n=64,split=2,split_mode=1,gather_warps=8" "split=4,split_mode=1" "split=4,split_mode=1,gather_warps=8"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py ns,ns_v32,gnmt50,gnmt75
done
for o in "persistent=2" "persistent=1" "persistent=1,gather_warps=8" "persistent=2,stages=2" "persistent=2,no_bulk_out=1"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py lf,ffn1,ffn2_v32
done
