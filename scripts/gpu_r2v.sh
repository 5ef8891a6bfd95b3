#!/bin/bash
cd $GRAFT_REPO_ROOT
for o in "split=0" "split=1" "split=4" "gather_warps=8" "split=2,gather_warps=8" "split=4,gather_warps=8" "persistent=2" "persistent=2,gather_warps=8" "stages=2" "stages=4"; do
echo "== $o"; SBW_OPTS=$o timeout 300 python scripts/ab_cases.py conv7,conv28,conv14
done
