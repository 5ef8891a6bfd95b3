#!/bin/bash
# NS family: cp.async hybrids / gather warps / unit shapes; LF ncu capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95
for o in tile_n=128 "tile_n=128,cp_async_slabs=1" "tile_n=128,cp_async_slabs=2" "tile_n=128,cp_async_slabs=1,split=2,split_mode=1" "tile_n=128,cp_async_slabs=2,split=4,split_mode=1" "tile_n=128,gather_warps=8" "tile_n=64,gather_warps=8" "tile_n=128,cp_async_slabs=1,split=4,split_mode=1" tile_n=128; do
  echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
done
python bench.py --workload lf --profile --steps 3 --warmup 1 --no-sharded > gpurun_out/lf_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm_persist -s 2 -c 1 -o gpurun_out/prof_lf_r2a python bench.py --workload lf --profile --steps 3 --warmup 1 --no-sharded > gpurun_out/ncu_lf.log 2>&1
tail -3 gpurun_out/ncu_lf.log
