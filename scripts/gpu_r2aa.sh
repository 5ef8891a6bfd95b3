#!/bin/bash
cd $GRAFT_REPO_ROOT
C=ns,ns_v32,gnmt50,ffn1,ffn1_50,ffn2_v32,lf
bash scripts/ab.sh "python scripts/ab_cases.py $C" paper_2203_05016_b200/lib/libshflbw_b200.so abl/SBW_NO_TILES.so
