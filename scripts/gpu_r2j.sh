#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -3 gpurun_out/tests.log
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95,attn128,ffn1_128,ffn2_128,ffn2,ffn1,ffn1_50,ffn2_v32
echo "== auto"; timeout 300 python scripts/ab_cases.py $C
echo "== gw8"; SBW_OPTS=gather_warps=8 timeout 300 python scripts/ab_cases.py $C
echo "== auto"; timeout 300 python scripts/ab_cases.py lf,conv56,conv28,conv14,conv7
for o in "split=0" "gather_warps=8"; do
echo "== trace $o"; SBW_LIB=$PWD/abl/trace.so timeout 120 python scripts/trace.py --chain 8 --opts $o 2>&1 | tail -26
done
