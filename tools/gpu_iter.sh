#!/bin/bash
# GPU call for kernel iteration: build, a parity subset (PYTEST_K), a short C4 bench, optional ncu
# of the kernels matching KREGEX.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout ${TEST_TIMEOUT:-420} python -m pytest tests -m gpu -x -q --timeout 300 -k "${PYTEST_K:-random or ragged or config_full or large_balls or errors or c3_full}" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
timeout ${BENCH_TIMEOUT:-420} python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.load(open("gpurun_out/bench.json"))
    print("ms/step", round(d["ms_per_step"], 3), "Gvox/s", round(d["value"], 2), "e2e", round(d["e2e"]["value"], 2))
    print({k: v["ms"] for k, v in d["stages"].items()})
except Exception as e:
    print("no bench json", e)
PY
if [ -n "$KREGEX" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$KREGEX" -o gpurun_out/prof_${TAG:-iter} -f python tools/prof_run.py --config ${CFG:-4} --iters 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
fi
