#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -2 gpurun_out/tests.log
for i in 1 2; do
echo "== auto"; timeout 300 python scripts/ab_cases.py ns,ffn1,ffn1_50,ffn2_v32,lf,conv56,conv28,c1x1_56,c1x1_14
done
