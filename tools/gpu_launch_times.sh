#!/bin/bash
# GPU call: per-kernel device times (ncu gpu__time_duration only) of one hot-path call.
mkdir -p gpurun_out
CMD="python tools/prof_run.py --config ${CFG:-4} --iters 1"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 $CMD > gpurun_out/lt_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lt_launches.csv $CMD > gpurun_out/lt_ncu.log 2>&1; echo "rc=$?"
python tools/launch_summary.py gpurun_out/lt_launches.csv
