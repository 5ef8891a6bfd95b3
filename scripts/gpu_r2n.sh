#!/bin/bash
cd $GRAFT_REPO_ROOT
for i in 1 2; do
echo "== auto"; timeout 300 python scripts/ab_cases.py ns,ffn1,ffn1_50,ffn2_v32,conv56,conv28,conv14,conv7,lf
done
