#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -15 gpurun_out/tests.log
for o in "gather_issue=0" "gather_issue=2" "gather_issue=0,tile_n=128" "gather_issue=0"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py ffn1,ffn1_50,ffn2_v32,conv56,conv28,conv14,conv7,lf
done
