cd $GRAFT_REPO_ROOT
SBW_TRACE=1 python -m paper_2203_05016_b200.build --force > gpurun_out/tr_build.log 2>&1 || { tail gpurun_out/tr_build.log; exit 1; }
for cfg in "--K 2048 --opts split=0" "--K 2048 --opts split=4,split_mode=2" "--K 256 --opts split=0" "--K 256 --opts split=1" "--K 256 --opts split=4,split_mode=2" "--K 8192 --opts split=0"; do
  timeout -k 10 120 python scripts/trace.py --chain 8 $cfg 2>&1 | tail -30
done > gpurun_out/trace.log
cat gpurun_out/trace.log
