cd $GRAFT_REPO_ROOT
timeout -k 10 300 python -m pytest tests/test_gpu_parity.py -x -q -k "split or ksplit" > gpurun_out/h_t.log 2>&1
echo "tests exit $?" >> gpurun_out/h_t.log
for K in 256 1024 2048 4096; do
timeout -k 10 120 python scripts/explore.py --workload ns --K $K --configs "split=0;split=4,split_mode=2;split=2,split_mode=1;split=4,split_mode=1" 2>&1 | tail -5
done > gpurun_out/h_ns.log
for V in 32 128; do
timeout -k 10 120 python scripts/explore.py --workload ns --V $V --configs "split=0;split=4,split_mode=2" 2>&1 | tail -3
done >> gpurun_out/h_ns.log
timeout -k 10 300 python scripts/explore.py --workload ns --M 4096 --K 1024 --configs "split=0;split=4,split_mode=2;split=2,split_mode=1" >> gpurun_out/h_ns.log 2>&1
tail -3 gpurun_out/h_t.log; cat gpurun_out/h_ns.log
