#!/bin/bash
# round-2 GPU check: microbench constants, the survivor/overflow tests, bench lines
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu && ./tools/microbench > gpurun_out/microbench.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_survivors.py -q > gpurun_out/t_surv.log 2>&1; tail -5 gpurun_out/t_surv.log
timeout 600 python bench.py > gpurun_out/b_cfg1.json 2> gpurun_out/b_cfg1.err; tail -c 400 gpurun_out/b_cfg1.err
timeout 600 python bench.py --config 0 > gpurun_out/b_cfg0.json 2> gpurun_out/b_cfg0.err; tail -c 400 gpurun_out/b_cfg0.err
timeout 900 python bench.py --config 2 --n 125000000 --steps 5 > gpurun_out/b_cfg2s.json 2> gpurun_out/b_cfg2s.err; tail -c 600 gpurun_out/b_cfg2s.err
