#!/bin/bash
# K6 ring v3 + bulk L2 prefetch of the next unit (main lib) vs v3 without it (tools/lib12/k6v3.so): parity, config-2 shape, config 4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/g35
O=gpurun_out/g35
timeout 1800 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_survivors.py -x -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -3 $O/pytest.log
for n in k6v3 new; do
  L=tools/lib12/$n.so; [ $n = new ] && L=paper_1609_01882_b200/libpoly_b200.so
  for np in 16 64; do
    POLY_B200_LIB=$L timeout 600 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 --nprobe $np 2>&1 | tail -1 | sed "s/^/$n np$np: /"
  done
  POLY_B200_LIB=$L timeout 900 python bench.py --config 4 --steps 10 --no-cpu-baseline --no-e2e > $O/cfg4_$n.json 2> $O/cfg4_$n.err; python -c "
import json
for l in open('$O/cfg4_$n.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$n cfg4 ms/step', d['ms_per_step'], 'codes/s', d['value'])"
  POLY_B200_LIB=$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_$n.csv python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 1 > $O/ncu_$n.log 2>&1
  python tools/launches.py $O/launch_$n.csv | grep -E "ivf_list_scan|total"
done
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:ivf_list_scan -s 1 -c 1 -o $O/k6_pf python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 1 > $O/ncu2.log 2>&1; echo "ncu k6 rc=$?"
