cd $GRAFT_REPO_ROOT
# One GPU call for a round's evidence: tests + smoke + bench lines, ncu launch
# lists and --set full captures of the SpMM kernels, the BASELINE sweep.
TAG=${1:-r1j}
bash scripts/gpu_round.sh > gpurun_out/round.log 2>&1
bash scripts/gpu_profile.sh ns $TAG > gpurun_out/profile_ns.log 2>&1
bash scripts/gpu_profile.sh ffn $TAG > gpurun_out/profile_ffn.log 2>&1
timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 2 -c 1 \
    -o gpurun_out/prof_lf_$TAG -f python bench.py --profile --workload lf --steps 4 --warmup 3 > gpurun_out/ncu_lf.log 2>&1
timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 20 -c 1 \
    -o gpurun_out/prof_conv56_$TAG -f python scripts/conv_profile.py > gpurun_out/ncu_conv.log 2>&1
timeout -k 10 900 python scripts/sweep.py --steps 300 --out gpurun_out/sweep > gpurun_out/sweep.log 2>&1
tail -5 gpurun_out/round.log; tail -n 3 gpurun_out/profile_ns.log gpurun_out/profile_ffn.log; tail -28 gpurun_out/sweep.log
