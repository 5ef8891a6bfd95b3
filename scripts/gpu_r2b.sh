#!/bin/bash
# Round-2: full GPU tests, then A/B of tile_n (64 vs 128) and raster (1 vs 2).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 1200 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -30 gpurun_out/tests.log
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95,attn128,ffn1_128,ffn2_128
for o in tile_n=128 tile_n=0 tile_n=128 tile_n=0; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
done
for o in raster=1 raster=2 raster=1 raster=2; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py lf,conv28,ffn1
done
timeout -k 10 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_drv.json 2> gpurun_out/bench_drv.err; echo "bench exit $?" >> gpurun_out/bench_drv.err
cat gpurun_out/bench_drv.json; tail -3 gpurun_out/bench_drv.err
