#!/bin/bash
# K6g (cell-major IVF scan): IVF parity + survivors, then cfg2 at the per-GPU share and 1e9 with batch 2048 / 10000
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_survivors.py -x -q > gpurun_out/t_ivf.log 2>&1; echo "ivf tests rc=$?"; tail -15 gpurun_out/t_ivf.log
for B in 2048 10000; do
timeout 900 python bench.py --config 2 --n 125000000 --batch $B --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg2s_$B.json 2> gpurun_out/b_cfg2s_$B.err; echo "cfg2s B=$B rc=$?"; tail -c 300 gpurun_out/b_cfg2s_$B.err
done
timeout 900 python bench.py --config 2 --batch 10000 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg2_10000.json 2> gpurun_out/b_cfg2_10000.err; echo "cfg2 B=10000 rc=$?"; tail -c 300 gpurun_out/b_cfg2_10000.err
