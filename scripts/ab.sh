#!/bin/bash
# A/B timing of library builds on one box (development): runs the command
# once per library, twice, alternating.   bash scripts/ab.sh "<cmd>" a.so b.so ...
cd $GRAFT_REPO_ROOT
CMD=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib (rep $rep)"
    SBW_LIB=$PWD/$lib timeout 300 bash -c "$CMD" 2>&1 | tail -40
  done
done
