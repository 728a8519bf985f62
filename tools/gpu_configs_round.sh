#!/bin/bash
# GPU call: every BASELINE config's device time, the C5 bench line, large objects, the slab path at one
# rank and the reference arm (TAG names the outputs).
mkdir -p gpurun_out
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python tools/all_configs.py > gpurun_out/all_configs_${TAG}.jsonl 2> gpurun_out/all_configs_${TAG}.err; echo "configs rc=$?"; tail -6 gpurun_out/all_configs_${TAG}.jsonl
timeout 600 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c5.json 2> gpurun_out/bench_${TAG}_c5.err; echo "c5 rc=$?"
timeout 900 python tools/large_objects.py > gpurun_out/large_objects_${TAG}.jsonl 2> gpurun_out/large_objects_${TAG}.err; echo "large rc=$?"; tail -6 gpurun_out/large_objects_${TAG}.jsonl
timeout 600 python bench.py --mode slab --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_slab1.json 2> gpurun_out/bench_${TAG}_slab1.err; echo "slab rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_${TAG}_reference.json 2> gpurun_out/bench_${TAG}_reference.err; echo "ref rc=$?"
