#!/bin/bash
# K6 ring v3 (dense row / code rings, lazy row read): IVF parity, A/B vs the kept K6 (base); ncu of K5t and of K6 v3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/g33
O=gpurun_out/g33
timeout 1500 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_survivors.py -x -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -3 $O/pytest.log
for n in base new; do
  L=tools/lib12/$n.so; [ $n = new ] && L=paper_1609_01882_b200/libpoly_b200.so
  for np in 16 64; do
    POLY_B200_LIB=$L timeout 600 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 --nprobe $np 2>&1 | tail -1 | sed "s/^/$n np$np: /"
  done
  POLY_B200_LIB=$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_$n.csv python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 1 > $O/ncu_$n.log 2>&1
  python tools/launches.py $O/launch_$n.csv | grep -E "ivf_list_scan|total"
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:ivf_list_scan -s 1 -c 1 -o $O/k6_ring3 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 1 > $O/ncu2.log 2>&1; echo "ncu k6 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coarse_tc -s 2 -c 1 -o $O/k5t python tools/prof_coarse.py --nq 10000 --reps 2 > $O/ncu3.log 2>&1; echo "ncu k5t rc=$?"
