#!/bin/bash
cd $GRAFT_REPO_ROOT
for i in 1 2; do
echo "== auto"; timeout 300 python scripts/ab_cases.py ns,ns_v32,ns_v128,gnmt50,ffn2_128,ffn2,ffn2_v32,conv7,lf
done
