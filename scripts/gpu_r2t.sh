#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout -k 10 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
tail -3 gpurun_out/tests.log
echo "== auto"; timeout 300 python scripts/ab_cases.py ns,ns_v32,gnmt50,ffn1,ffn1_50,ffn2,lf,conv56
timeout 600 python scripts/compare_formats.py --out gpurun_out/formats_r2 > gpurun_out/formats.log 2>&1; tail -12 gpurun_out/formats_r2.md
