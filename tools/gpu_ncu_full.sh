#!/bin/bash
# GPU call: one ncu --set full capture of every hot-path kernel of one C4 call.
mkdir -p gpurun_out
CMD="python tools/prof_run.py --config ${CFG:-4} --iters 1"
timeout 600 $CMD > gpurun_out/prof_plain.log 2>&1 && timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_(edt|prune|dilate)}" -s ${SKIP:-6} -c ${COUNT:-6} -o gpurun_out/prof_${TAG:-c4} -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/ncu_full.log
