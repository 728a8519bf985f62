#!/bin/bash
# GPU call: gpu tests + a short C4 bench without the CPU baseline.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-420} python -m pytest tests -m gpu -x -q --durations=6 --timeout 300 ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/gpu_tests.log
timeout ${BENCH_TIMEOUT:-420} python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
