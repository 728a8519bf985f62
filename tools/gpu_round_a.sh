#!/bin/bash
# GPU call A: build, smoke, gpu tests, bench (C4 with the CPU baseline), slab-mode bench at N=1,
# and the ncu launch list of a short bench run.
mkdir -p gpurun_out
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc; lscpu | grep -E "Model name|^CPU\(s\)"; } > gpurun_out/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { echo SMOKE FAILED; tail -30 gpurun_out/smoke.log; }
tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q --durations=8 --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --mode slab --steps 3 --warmup 3 > gpurun_out/bench_slab.json 2> gpurun_out/bench_slab.err; echo "slab bench rc=$?"; cat gpurun_out/bench_slab.json; tail -3 gpurun_out/bench_slab.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
