#!/bin/bash
# Evidence for profiles/: plain bench, ncu launch list of the same command, one
# full-set capture of the main K2 launch (cold-cache, serialized: compare shares).
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --per-ht 28,32 --no-cpu-baseline"
$CMD > gpurun_out/plain_bench.json 2> gpurun_out/plain_bench.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch-list rc=$?"
C2="python tools/prof_scan.py --n 100000000 --ht 24"
$C2 > gpurun_out/plain_scan.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 0 -c 1 -o gpurun_out/prof_scan_full $C2 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
