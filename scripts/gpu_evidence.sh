cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_round.sh > gpurun_out/round.log 2>&1
timeout -k 10 900 python scripts/sweep.py --steps 300 --out gpurun_out/sweep > gpurun_out/sweep.log 2>&1
bash scripts/gpu_profile.sh ns r1l > gpurun_out/profile_ns.log 2>&1
tail -4 gpurun_out/round.log; cat gpurun_out/sweep.md; tail -2 gpurun_out/profile_ns.log
