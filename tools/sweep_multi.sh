#!/bin/bash
# GPU call: C4 bench per compile-time configuration (edit the list).
mkdir -p gpurun_out
for cfg in "" "-DFASTRS_COL_STATIC"; do
  FASTRS_NVCC_DEFS="$cfg" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build $cfg failed"; continue; }
  timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d = json.load(open('gpurun_out/sw.json'))
print('$cfg', round(d['ms_per_step'], 3), {k: v['ms'] for k, v in d['stages'].items()})"
done
