cd $GRAFT_REPO_ROOT
timeout -k 10 300 python -m pytest tests/test_gpu_parity.py -q -x -k "split or ksplit or persistent or tc_matches" > gpurun_out/ns_t.log 2>&1; tail -2 gpurun_out/ns_t.log
timeout -k 10 300 python scripts/explore.py --workload ns --configs "split=0;split=4,split_mode=3;split=4,split_mode=1" 2>&1 | tail -4
timeout -k 10 300 python scripts/opt_sweep.py --opts "persistent=0" --only "FFN,large,GNMT 4096x1024 N=128 75" 2>&1 | grep "{"
SBW_TRACE=1 python -m paper_2203_05016_b200.build --force > gpurun_out/tr_build.log 2>&1 && timeout -k 10 120 python scripts/trace.py --chain 8 --K 2048 2>&1 | tail -12
