cd $GRAFT_REPO_ROOT
C="split=0;split=4,split_mode=2,cp_async_slabs=1;split=4,split_mode=2,cp_async_slabs=2;split=4,split_mode=2,cp_async_slabs=1,stages=6;split=4,split_mode=3;split=4,split_mode=3,cp_async_slabs=1;split=4,split_mode=1,cp_async_slabs=1;split=1,cp_async_slabs=1;split=1,cp_async_slabs=2"
for K in 2048 4096; do
timeout -k 10 200 python scripts/explore.py --workload ns --K $K --configs "$C" 2>&1 | tail -10
done > gpurun_out/cps.log
timeout -k 10 200 python scripts/explore.py --workload ffn --configs "split=0;split=0,cp_async_slabs=1;split=0,cp_async_slabs=2" >> gpurun_out/cps.log 2>&1
cat gpurun_out/cps.log
