#!/bin/bash
# lean K6 (item mode, G = 1) and cell mode (G = 4): parity, timings at the cfg2 per-GPU share, cfg2 at 1e9
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_survivors.py -x -q > gpurun_out/t_ivf.log 2>&1; echo "ivf tests rc=$?"; tail -5 gpurun_out/t_ivf.log
bash tools/build_variant.sh cell -DPOLY_IVF_CELL=1 > /dev/null 2>&1 || echo "variant build failed"
POLY_B200_LIB=tools/lib12/cell.so timeout 900 python -m pytest tests/test_gpu_ivf.py -x -q -k "randomized or larger or knn" > gpurun_out/t_ivf_cell.log 2>&1; echo "cell-mode ivf tests rc=$?"; tail -3 gpurun_out/t_ivf_cell.log
for v in default cell; do
  L=""; [ $v != default ] && L=tools/lib12/$v.so
  for nq in 2048 10000; do
    POLY_B200_LIB=$L timeout 600 python tools/prof_ivf.py --n 125000000 --nq $nq --batch $nq --reps 3 2>&1 | tail -1 | sed "s/^/$v nq=$nq: /"
  done
done
for B in 2048 10000; do
timeout 900 python bench.py --config 2 --batch $B --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/b_cfg2_k6l_$B.json 2> gpurun_out/b_cfg2_k6l_$B.err; echo "cfg2 B=$B rc=$?"; tail -c 300 gpurun_out/b_cfg2_k6l_$B.err
done
