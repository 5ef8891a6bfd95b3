#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -3 gpurun_out/tests.log
C=ns,ns_v32,ns_v128,gnmt50,gnmt75,gnmt95,attn128,ffn1_128,ffn2_128,ffn2,ffn1,ffn1_50,ffn2_v32
echo "== auto"; timeout 300 python scripts/ab_cases.py $C
echo "== auto"; timeout 300 python scripts/ab_cases.py lf,conv56,conv28,conv14,conv7
python bench.py --profile --steps 200 --warmup 10 --no-sharded > gpurun_out/ns_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm_tc -s 50 -c 1 -o gpurun_out/prof_ns_r2a python bench.py --profile --steps 200 --warmup 10 --no-sharded > gpurun_out/ncu_ns.log 2>&1
tail -2 gpurun_out/ncu_ns.log
