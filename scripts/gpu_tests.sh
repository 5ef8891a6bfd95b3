cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout -k 10 200 python -m pytest tests/test_gpu_parity.py -x -q -k "known_answers or random_sequences or unit_instances" > gpurun_out/t1.log 2>&1
echo "t1 exit $?" >> gpurun_out/t1.log
timeout -k 10 600 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/t2.log 2>&1
echo "t2 exit $?" >> gpurun_out/t2.log
tail -5 gpurun_out/t1.log; tail -30 gpurun_out/t2.log
