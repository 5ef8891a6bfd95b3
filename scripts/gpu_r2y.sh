#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -3 gpurun_out/tests.log
for o in "xchg_bulk=0" "xchg_bulk=-1" "xchg_bulk=0" "xchg_bulk=-1"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py ns,ns_v32,ns_v128,gnmt50,ffn2_128,ffn2,ffn2_v32,conv7
done
