cd $GRAFT_REPO_ROOT
for K in 256 512 1024 2048 4096 8192; do
timeout -k 10 120 python scripts/explore.py --workload ns --K $K --configs "split=0;split=1;split=4,split_mode=2" 2>&1 | tail -4
done > gpurun_out/scan_k.log
for M in 512 1024 4096; do
timeout -k 10 120 python scripts/explore.py --workload ns --M $M --configs "split=0" 2>&1 | tail -2
done > gpurun_out/scan_m.log
cat gpurun_out/scan_k.log gpurun_out/scan_m.log
