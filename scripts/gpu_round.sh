#!/bin/bash
# One GPU call: parity tests, smoke, bench, then an ncu launch list of the bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
timeout -k 10 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout -k 10 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout -k 10 300 python bench.py --workload ffn --no-cpu-baseline > gpurun_out/bench_ffn.json 2>> gpurun_out/bench.err
tail -3 gpurun_out/tests.log; cat gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err; cat gpurun_out/bench_ffn.json
