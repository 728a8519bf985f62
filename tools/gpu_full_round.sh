#!/bin/bash
# GPU call: gpu tests + smoke, then the profile round (bench + launch list + ncu --set full), TAG names it.
mkdir -p gpurun_out
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q --durations=6 --timeout 400 ${PYTEST_ARGS} > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo "tests rc=$?"; tail -12 gpurun_out/gpu_tests_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_${TAG}.log
TAG=$TAG bash tools/gpu_profile_round.sh
