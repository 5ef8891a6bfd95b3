#!/bin/bash
# ncu evidence for one workload: a plain run first (must exit 0), then the
# launch list and one --set full capture of the SpMM kernel.
#   bash scripts/gpu_profile.sh <workload> <tag>
cd $GRAFT_REPO_ROOT
WL=${1:-ns}; TAG=${2:-r1}
mkdir -p gpurun_out
CMD="python bench.py --profile --workload $WL --steps 40 --warmup 4"
$CMD > gpurun_out/plain_$WL.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${WL}_${TAG}.csv $CMD > gpurun_out/ncu_launch_$WL.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 8 -c 1 -o gpurun_out/prof_${WL}_${TAG} -f $CMD > gpurun_out/ncu_full_$WL.log 2>&1
echo "exit $?"
tail -n 3 gpurun_out/plain_$WL.log gpurun_out/ncu_full_$WL.log
