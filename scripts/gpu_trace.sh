cd $GRAFT_REPO_ROOT
SBW_TRACE=1 python -m paper_2203_05016_b200.build --force > gpurun_out/tr_build.log 2>&1 || { tail gpurun_out/tr_build.log; exit 1; }
timeout -k 10 120 python scripts/trace.py --chain 8 --K 2048 2>&1 | tail -32 > gpurun_out/ns_trace.log
cat gpurun_out/ns_trace.log
