#!/bin/bash
# round-2 evidence: cfg4 with the full 1e7-row graph through the file sink, cfg0, cfg3 lines; ncu of the m = 16 K2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python bench.py --config 4 --steps 10 --knn-full /tmp/knn_full.knng > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err; echo "cfg4 rc=$?"; tail -c 300 gpurun_out/b_cfg4.err
timeout 600 python bench.py --config 0 > gpurun_out/b_cfg0.json 2> gpurun_out/b_cfg0.err; echo "cfg0 rc=$?"; tail -c 300 gpurun_out/b_cfg0.err
timeout 1200 python bench.py --config 3 --steps 5 > gpurun_out/b_cfg3.json 2> gpurun_out/b_cfg3.err; echo "cfg3 rc=$?"; tail -c 300 gpurun_out/b_cfg3.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_kernel -c 1 -o gpurun_out/r02_k2_m16 python tools/prof_scan.py --m 16 --n 50000000 --ht 56 > gpurun_out/ncu_k2m16.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_k2m16.log
