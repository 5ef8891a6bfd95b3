#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -5 gpurun_out/tests.log
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95,attn128,ffn1_128,ffn2_128,ffn2,ffn1,ffn1_50,ffn2_v32
for o in "nacc=1,tile_n=128" "tile_n=128" "nacc=4,tile_n=128" "nacc=1,tile_n=64" "tile_n=64" "nacc=4,tile_n=64"; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
done
for o in "nacc=1" "nacc=0" "nacc=4"; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py lf,conv56,conv28,conv14,conv7
done
for o in "tile_n=128,nacc=1" "tile_n=128,nacc=4"; do
  echo "== trace $o"; SBW_LIB=$PWD/abl/trace.so timeout 120 python scripts/trace.py --chain 8 --opts $o 2>&1 | tail -22
done
