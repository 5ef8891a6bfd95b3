#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -3 gpurun_out/tests.log
for o in "stages=0" "stages=3" "stages=0"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py lf,ffn1,ffn1_50,ffn2_v32,conv56,conv28,ffn2
done
