#!/bin/bash
# Round-2: targeted tests + NS unit-shape A/B + traces + LF raster A/B.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests -m gpu -q -k "half_width or persistent_kernel_bitwise or raster or auto_plan" > gpurun_out/tests_c.log 2>&1; echo "tests exit $?" >> gpurun_out/tests_c.log
tail -15 gpurun_out/tests_c.log
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95,attn128,ffn1_128,ffn2_128
for o in tile_n=128 tile_n=64 "tile_n=64,split=4,split_mode=1" "tile_n=64,split=2,split_mode=3" "tile_n=64,split=1,split_mode=3" "tile_n=64,split=4,split_mode=2" tile_n=128 tile_n=64; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
done
for o in raster=1 raster=2 raster=1 raster=2; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py lf,conv28,ffn1
done
for o in tile_n=128 tile_n=64 "tile_n=64,split=4,split_mode=1"; do
  echo "== trace $o"; SBW_LIB=$PWD/abl/trace.so timeout 120 python scripts/trace.py --chain 8 --opts $o 2>&1 | tail -40
done
