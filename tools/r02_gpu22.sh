#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:ivf_list_scan -s 1 -c 1 -o gpurun_out/r02_k6_r2_4e8 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 1 > gpurun_out/ncu_k6r2.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_k6r2.log
