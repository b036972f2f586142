#!/bin/bash
# Second evidence pass: launch lists of configs 0 / 3 / 4, the 8-rank by-list emulation (config 2, 1e9 codes), microbench constants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/evidence2
O=gpurun_out/evidence2
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_cfg4.csv env BENCH_PROFILE=1 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu4.log 2>&1; echo "ncu4=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_cfg3.csv env BENCH_PROFILE=1 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --per-ht "" > $O/ncu3.log 2>&1; echo "ncu3=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_cfg0.csv env BENCH_PROFILE=1 python bench.py --config 0 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --per-ht "" > $O/ncu0.log 2>&1; echo "ncu0=$?"
timeout 2400 python tools/emulate_bylist.py > $O/emulate_bylist_rank0of8.json 2> $O/emulate.err; echo "emulate rc=$?"; tail -1 $O/emulate_bylist_rank0of8.json | cut -c1-600
