#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 600 python -m pytest tests/test_sharded.py -m gpu -q -rs > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -8 gpurun_out/tests.log
nvidia-smi -q | grep -i -A2 "fabric\|multicast" | head -20
