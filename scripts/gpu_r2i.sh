#!/bin/bash
cd $GRAFT_REPO_ROOT
for o in "split=0" "tile_n=64,split=1,split_mode=3"; do
  echo "== trace $o"; SBW_LIB=$PWD/abl/trace.so timeout 120 python scripts/trace.py --chain 8 --opts $o 2>&1 | tail -26
done
echo "== warm"; SBW_WARM=1 SBW_LIB=$PWD/abl/trace.so timeout 120 python scripts/trace.py --chain 8 2>&1 | tail -26
