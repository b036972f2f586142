#!/bin/bash
# K5t stages: 4 x 32 KB (k6v3.so) vs 5 x 32 KB (main) vs 10 x 16 KB (k16.so); coarse + k-means parity on the main build
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/g37
O=gpurun_out/g37
for n in k6v3 new k16; do
  L=tools/lib12/$n.so; [ $n = new ] && L=paper_1609_01882_b200/libpoly_b200.so
  POLY_B200_LIB=$L timeout 600 python tools/prof_coarse.py --nq 10000 --reps 5 2>&1 | tail -1 | sed "s/^/$n d128: /"
  POLY_B200_LIB=$L timeout 600 python tools/prof_coarse.py --nq 2048 --nlist 16384 --dim 256 --nprobe 32 --reps 5 2>&1 | tail -1 | sed "s/^/$n d256: /"
  POLY_B200_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:coarse_ --csv --log-file $O/launch_$n.csv python tools/prof_coarse.py --nq 10000 --reps 1 > $O/ncu_$n.log 2>&1
  python tools/launches.py $O/launch_$n.csv | tail -3
done
timeout 1800 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_kmeans.py -x -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -3 $O/pytest.log
POLY_B200_LIB=tools/lib12/k16.so timeout 1800 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_kmeans.py -x -q > $O/pytest_k16.log 2>&1; echo "tests k16 rc=$?"; tail -3 $O/pytest_k16.log
