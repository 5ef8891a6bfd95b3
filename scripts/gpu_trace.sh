cd $GRAFT_REPO_ROOT
SBW_TRACE=1 python -m paper_2203_05016_b200.build --force > gpurun_out/tr_build.log 2>&1 || { tail gpurun_out/tr_build.log; exit 1; }
for cfg in "--workload conv56 --prepared --opts persistent=-1" "--workload conv56 --prepared --opts persistent=2 --persist" "--workload conv14 --prepared --opts persistent=-1"; do
  timeout -k 10 120 python scripts/conv_trace.py --chain 4 $cfg 2>&1 | tail -32
done > gpurun_out/conv_trace.log
cat gpurun_out/conv_trace.log
