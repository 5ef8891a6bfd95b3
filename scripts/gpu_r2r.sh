#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x -k "persistent or large_ffn or raster or deep" > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -3 gpurun_out/tests.log
for o in "prefetch_next=0" "prefetch_next=-1" "prefetch_next=0" "prefetch_next=-1"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py lf,ffn1,ffn1_50,ffn2_v32,conv56
done
