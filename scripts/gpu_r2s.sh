#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x -k "async or compress" > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -15 gpurun_out/tests.log
timeout 300 python scripts/compress_probe.py
