#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95,attn128,ffn1_128,ffn2_128,ffn2
for o in "prefetch=0,tile_n=128" "prefetch=1,tile_n=128" "prefetch=1,tile_n=64" "prefetch=1,tile_n=64,split=4,split_mode=1" "prefetch=1,tile_n=128,split=4,split_mode=1" "prefetch=0,tile_n=128" "prefetch=1,tile_n=128"; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
done
for o in "prefetch=1,tile_n=128" "prefetch=1,tile_n=64"; do
  echo "== trace $o"; SBW_LIB=$PWD/abl/trace.so timeout 120 python scripts/trace.py --chain 8 --opts $o 2>&1 | tail -24
done
for o in persistent=2 persistent=1 "persistent=1,gather_warps=8"; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py lf
done
