#!/bin/bash
# GPU round trip used during development: parity tests, then the default bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
    print("value %.3e  ms/step %.2f  e2e %.3e  issue-frac %.3f" % (d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline_issue"]["frac"]))
    print({k: round(v["ms_per_step"], 2) for k, v in d["per_ht"].items()})
except Exception as e:
    print("no bench line", e)
PY
