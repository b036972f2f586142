#!/bin/bash
# after: K2 pair flush, K5t grid fill, K6 round-1 pre-selection -- full GPU suite, cfg1, cfg2 (1e9) + launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu_all.log 2>&1; echo "gpu suite rc=$?"; tail -6 gpurun_out/t_gpu_all.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b_cfg1_pair.json 2> gpurun_out/b_cfg1_pair.err; echo "cfg1 rc=$?"; tail -c 300 gpurun_out/b_cfg1_pair.err
timeout 1500 python bench.py --config 2 --steps 5 --no-cpu-baseline > gpurun_out/b_cfg2_v2.json 2> gpurun_out/b_cfg2_v2.err; echo "cfg2 rc=$?"; tail -c 300 gpurun_out/b_cfg2_v2.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launch_cfg2_1e9_v2.csv env BENCH_PROFILE=1 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --per-nprobe "" > gpurun_out/ncu_cfg2.log 2>&1; echo ncu=$?
