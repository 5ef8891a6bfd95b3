#!/bin/bash
cd $GRAFT_REPO_ROOT
for o in "probe=0" "probe=1" "probe=0" "probe=1"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py ns,ns_v32,gnmt50
done
