#!/bin/bash
# K5t: where the remaining time goes (timing-only variant without the selection network; ncu of the kept kernel); full GPU suite on the build
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/g36
O=gpurun_out/g36
for n in noepi new; do
  L=tools/lib12/$n.so; [ $n = new ] && L=paper_1609_01882_b200/libpoly_b200.so
  POLY_B200_LIB=$L timeout 600 python tools/prof_coarse.py --nq 10000 --reps 5 2>&1 | tail -1 | sed "s/^/$n coarse: /"
  POLY_B200_LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:coarse_ --csv --log-file $O/launch_$n.csv python tools/prof_coarse.py --nq 10000 --reps 1 > $O/ncu_$n.log 2>&1
  python tools/launches.py $O/launch_$n.csv | tail -4
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coarse_tc -s 2 -c 1 -o $O/k5t_new python tools/prof_coarse.py --nq 10000 --reps 2 > $O/ncu3.log 2>&1; echo "ncu k5t rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -3 $O/pytest.log
