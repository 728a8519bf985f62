#!/bin/bash
# GPU call: rebuild with each value of a compile-time knob and run the C4 bench (tuning sweeps).
# usage: MACRO=FASTRS_KPOINT VALUES="64 96 128" bash tools/sweep_define.sh
mkdir -p gpurun_out
for v in ${VALUES}; do
  FASTRS_NVCC_DEFS="-D${MACRO}=${v}" python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$v.log 2>&1 || { echo "build $v failed"; tail -5 gpurun_out/build_$v.log; continue; }
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/sweep_${MACRO}_$v.json 2>/dev/null
  python -c "
import json; d = json.load(open('gpurun_out/sweep_${MACRO}_$v.json'))
print('${MACRO}=$v', round(d['ms_per_step'], 3), {k: v['ms'] for k, v in d['stages'].items()})"
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
