#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,attn128,ffn2_128,ffn2
for o in "prefetch=0" "prefetch=2" "prefetch=0,tile_n=64" "prefetch=2,tile_n=64"; do
  echo "== cold $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
  echo "== warm $o"; SBW_WARM=1 SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
done
for o in "prefetch=0" "prefetch=2"; do
  echo "== trace cold $o"; SBW_LIB=$PWD/abl/trace.so timeout 120 python scripts/trace.py --chain 8 --opts $o 2>&1 | tail -22
done
echo "== trace warm"; SBW_WARM=1 SBW_LIB=$PWD/abl/trace.so timeout 120 python scripts/trace.py --chain 8 --opts prefetch=0 2>&1 | tail -22
