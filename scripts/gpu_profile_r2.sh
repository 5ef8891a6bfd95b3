#!/bin/bash
# Round-2 evidence: driver-style bench, default bench, ncu launch list and
# full captures of the north-star / large-FFN / FFN2 kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2a}
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks_$T.csv &
SMI=$!
timeout -k 10 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_drv_$T.json 2> gpurun_out/bench_drv_$T.err
timeout -k 10 900 python bench.py > gpurun_out/bench_full_$T.json 2> gpurun_out/bench_full_$T.err
timeout -k 10 600 python bench.py --workload lf --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_lf_$T.json 2>> gpurun_out/bench_full_$T.err
kill $SMI
P="python bench.py --profile --steps 20 --warmup 5 --no-sharded"
$P > gpurun_out/p_ns.log 2>&1 && $P --workload lf > gpurun_out/p_lf.log 2>&1 && $P --workload ffn > gpurun_out/p_ffn.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_ns_$T.csv $P > gpurun_out/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 10 -c 1 -o gpurun_out/prof_ns_$T $P > gpurun_out/ncu_ns.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/prof_lf_$T $P --workload lf > gpurun_out/ncu_lf.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 10 -c 1 -o gpurun_out/prof_ffn_$T $P --workload ffn > gpurun_out/ncu_ffn.log 2>&1
echo "ncu rc $?"
# converter: warm timings, launch list, full captures of the large-FFN pack / plan / pack kernels
python scripts/compress_probe.py > gpurun_out/compress_probe_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_conv_$T.csv python scripts/compress_kernels.py > gpurun_out/ncu_conv_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_pack_rows16|k_pack_group|k_plan" -s 6 -c 3 -o gpurun_out/prof_conv_$T python scripts/compress_kernels.py > gpurun_out/ncu_conv.log 2>&1
echo "ncu conv rc $?"
# reports -> csv pages (the .ncu-rep files would overflow the 64 MiB return)
for r in gpurun_out/prof_*_$T.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > ${b}_raw.csv 2>/dev/null
  ncu -i $r --page details --csv > ${b}_details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass 2>/dev/null | gzip > ${b}_source.csv.gz
  rm -f $r
done
ls -la gpurun_out | tail -20
cat gpurun_out/bench_drv_$T.json; tail -3 gpurun_out/bench_drv_$T.err
