#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ivf.py -x -q -k "by_list or sharded" > gpurun_out/t_bylist.log 2>&1; echo "bylist tests rc=$?"; tail -15 gpurun_out/t_bylist.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu_all.log 2>&1; echo "gpu suite rc=$?"; tail -4 gpurun_out/t_gpu_all.log
