#!/bin/bash
# K2 with the bias preloaded (2 MMAs per 128 codes): flat parity + cfg1
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_survivors.py tests/test_gpu_sharded.py -x -q > gpurun_out/t_flat.log 2>&1; echo "flat tests rc=$?"; tail -3 gpurun_out/t_flat.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b_cfg1_dbias.json 2> gpurun_out/b_cfg1_dbias.err; echo "cfg1 rc=$?"; tail -c 300 gpurun_out/b_cfg1_dbias.err
