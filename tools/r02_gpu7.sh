#!/bin/bash
# ncu --set full of one K2t launch (N = 1e8, 256 queries, ht 24)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_tc_kernel -c 1 -o gpurun_out/r02_k2t python tools/prof_scan.py --n 100000000 --ht 24 > gpurun_out/ncu_k2t.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_k2t.log
