#!/bin/bash
# ncu of the lean K6 (round-2 launch) at the cfg2 single-GPU size (1e9 codes), 2048 queries
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:ivf_list_scan -s 1 -c 1 -o gpurun_out/r02_k6lean_1e9 python tools/prof_ivf.py --n 400000000 --nq 2048 --batch 2048 --reps 1 > gpurun_out/ncu_k6lean.log 2>&1; echo ncu=$?; tail -3 gpurun_out/ncu_k6lean.log
