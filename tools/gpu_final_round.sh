#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r02k}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --durations=6 --timeout 400 > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --mode slab --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_slab1.json 2> gpurun_out/bench_${TAG}_slab1.err; echo "slab rc=$?"; head -c 600 gpurun_out/bench_${TAG}_slab1.json; tail -5 gpurun_out/bench_${TAG}_slab1.err
