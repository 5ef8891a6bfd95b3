#!/bin/bash
cd $GRAFT_REPO_ROOT
for o in "no_bulk_out=0" "no_bulk_out=1" "no_bulk_out=0" "no_bulk_out=1"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py ns,ns_v32,ns_v128,gnmt50,gnmt75,attn128,ffn2_128
done
