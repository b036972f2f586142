#!/bin/bash
# K6 (item-major) vs K6g (cell-major) at the cfg2 per-GPU share: timings + ncu of the round-2 scan
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/t_sharded.log 2>&1; echo "sharded tests rc=$?"; tail -15 gpurun_out/t_sharded.log
bash tools/build_variant.sh k6old -DPOLY_IVF_CELL=0 > /dev/null 2>&1 || echo "variant build failed"
for v in k6old default; do
  L=""; [ $v != default ] && L=tools/lib12/$v.so
  for nq in 2048 10000; do
    POLY_B200_LIB=$L timeout 600 python tools/prof_ivf.py --n 125000000 --nq $nq --batch $nq --reps 3 2>&1 | tail -1 | sed "s/^/$v nq=$nq: /"
  done
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:ivf_cell_scan -s 1 -c 1 -o gpurun_out/r02_k6g_b2048 python tools/prof_ivf.py --n 125000000 --nq 2048 --batch 2048 --reps 1 > gpurun_out/ncu_k6g.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:ivf_cell_scan -s 1 -c 1 -o gpurun_out/r02_k6g_b10000 python tools/prof_ivf.py --n 125000000 --nq 10000 --batch 10000 --reps 1 > gpurun_out/ncu_k6g2.log 2>&1; echo ncu2=$?
