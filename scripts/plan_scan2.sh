#!/bin/bash
# Development: cluster-split and persistence variants over the BASELINE cases.
cd $GRAFT_REPO_ROOT
C=ns,ns_v32,ns_v128,attn128,ffn1_128,ffn2_128,attn4096,ffn1,ffn1_50,ffn1_90,ffn2,ffn2_v32,ffn2_v128,gnmt50,gnmt75,gnmt90,gnmt95,conv56,conv28,conv14,conv7,c1x1_56,c1x1_14
for o in split=0 split=1 split=2,split_mode=1 split=2,split_mode=3 split=4,split_mode=1 split=4,split_mode=2 split=4,split_mode=3 persistent=-1 persistent=1 persistent=2 split=0; do
  echo "== $o"
  SBW_OPTS=$o timeout 300 python scripts/ab_cases.py $C 2>&1 | grep '^{'
done
