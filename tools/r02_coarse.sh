#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_ivf.py -x -q -k "probe_order" > gpurun_out/t_probe.log 2>&1; tail -15 gpurun_out/t_probe.log
timeout 900 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_survivors.py -x -q > gpurun_out/t_ivf.log 2>&1; tail -15 gpurun_out/t_ivf.log
timeout 900 python bench.py --config 2 --n 125000000 --steps 5 --no-cpu-baseline > gpurun_out/b_cfg2s.json 2> gpurun_out/b_cfg2s.err; tail -c 600 gpurun_out/b_cfg2s.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launch_cfg2s.csv env BENCH_PROFILE=1 python bench.py --config 2 --n 125000000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --per-nprobe "" > /dev/null 2>&1; echo ncu=$?
