#!/bin/bash
# Round-2 GPU call: parity tests (all -m gpu), smoke, the default bench, the
# driver-style short bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -k 10 1200 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/tests.log
timeout -k 10 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout -k 10 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_drv.json 2> gpurun_out/bench_drv.err; echo "bench exit $?" >> gpurun_out/bench_drv.err
timeout -k 10 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2>> gpurun_out/bench_drv.err
tail -25 gpurun_out/tests.log; cat gpurun_out/smoke.log; cat gpurun_out/bench_drv.json; tail -5 gpurun_out/bench_drv.err; cat gpurun_out/bench_ref.json
