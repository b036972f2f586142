#!/bin/bash
# cfg2 at 1e9 (one step = all 10,000 queries) full line; by-list build path at world 1; launch list at 1e9
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python bench.py --config 2 --steps 5 > gpurun_out/b_cfg2_full.json 2> gpurun_out/b_cfg2_full.err; echo "cfg2 rc=$?"; tail -c 300 gpurun_out/b_cfg2_full.err
timeout 900 python bench.py --config 2 --n 125000000 --ivf-shard list --steps 3 --no-cpu-baseline --no-e2e --per-nprobe "" > gpurun_out/b_cfg2_bylist.json 2> gpurun_out/b_cfg2_bylist.err; echo "bylist rc=$?"; tail -c 300 gpurun_out/b_cfg2_bylist.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/r02_launch_cfg2_1e9.csv env BENCH_PROFILE=1 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --per-nprobe "" > gpurun_out/ncu_cfg2.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_cfg2.log
