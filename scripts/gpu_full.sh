cd $GRAFT_REPO_ROOT
bash scripts/gpu_round.sh > gpurun_out/round.log 2>&1
bash scripts/gpu_profile.sh ns r1h > gpurun_out/profile_ns.log 2>&1
bash scripts/gpu_profile.sh ffn r1h > gpurun_out/profile_ffn.log 2>&1
timeout -k 10 900 python scripts/sweep.py --steps 300 --out gpurun_out/sweep > gpurun_out/sweep.log 2>&1
tail -5 gpurun_out/round.log; tail -3 gpurun_out/profile_ns.log gpurun_out/profile_ffn.log; tail -28 gpurun_out/sweep.log
