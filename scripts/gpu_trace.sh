cd $GRAFT_REPO_ROOT
SBW_TRACE=1 python -m paper_2203_05016_b200.build --force > gpurun_out/tr_build.log 2>&1 || { tail gpurun_out/tr_build.log; exit 1; }
for cfg in "--workload ffn --opts persistent=1 --persist" "--workload ffn --opts persistent=-1" "--workload lf --opts persistent=1 --persist"; do
  timeout -k 10 200 python scripts/trace.py $cfg 2>&1 | tail -40
done > gpurun_out/ptrace.log
cat gpurun_out/ptrace.log
