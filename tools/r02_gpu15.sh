#!/bin/bash
# IVF suites after the K1r item lists / split change; by-list sharding; full gpu suite
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu_all.log 2>&1; echo "gpu suite rc=$?"; tail -8 gpurun_out/t_gpu_all.log
timeout 900 python bench.py --config 2 --n 125000000 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg2s.json 2> gpurun_out/b_cfg2s.err; echo "cfg2s rc=$?"; tail -c 300 gpurun_out/b_cfg2s.err
timeout 900 python bench.py --config 4 --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg4b.json 2> gpurun_out/b_cfg4b.err; echo "cfg4 rc=$?"; tail -c 300 gpurun_out/b_cfg4b.err
