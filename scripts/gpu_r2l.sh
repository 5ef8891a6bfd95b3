#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -3 gpurun_out/tests.log
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95,attn128,ffn1_128,ffn2_128,ffn2,ffn1,ffn1_50,ffn2_v32
for o in "gather_issue=0" "gather_issue=2" "gather_issue=0"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py lf,conv28,conv14
done
