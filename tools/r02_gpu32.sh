#!/bin/bash
# K6 ring + unit prefetch: IVF parity, A/B vs the previous K6 (base) and a 12-CTA/SM build
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/g32
O=gpurun_out/g32
timeout 1500 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_survivors.py -x -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -3 $O/pytest.log
for n in base new new12; do
  L=tools/lib12/$n.so; [ $n = new ] && L=paper_1609_01882_b200/libpoly_b200.so
  POLY_B200_LIB=$L timeout 600 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 --nprobe 16 2>&1 | tail -1 | sed "s/^/$n np16: /"
  POLY_B200_LIB=$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_$n.csv python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 1 > $O/ncu_$n.log 2>&1
  python tools/launches.py $O/launch_$n.csv | grep -E "ivf_list_scan|total"
done
