#!/bin/bash
# round-2 GPU pass 1: full gpu suite, smoke, cfg1/cfg0/cfg2 bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/b_cfg1.json 2> gpurun_out/b_cfg1.err; echo "cfg1 rc=$?"; tail -c 300 gpurun_out/b_cfg1.err
timeout 900 python bench.py --config 2 --steps 5 > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err; echo "cfg2 rc=$?"; tail -c 600 gpurun_out/b_cfg2.err
