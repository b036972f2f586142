#!/bin/bash
# Branch-free K5t epilogue + K6 ring v3: IVF / k-means / survivor parity, coarse timing, config-2 shape and config 4 A/B vs base
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/g34
O=gpurun_out/g34
timeout 1800 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_survivors.py tests/test_gpu_kmeans.py -x -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -3 $O/pytest.log
for n in base new; do
  L=tools/lib12/$n.so; [ $n = new ] && L=paper_1609_01882_b200/libpoly_b200.so
  POLY_B200_LIB=$L timeout 600 python tools/prof_coarse.py --nq 10000 --reps 5 2>&1 | tail -1 | sed "s/^/$n coarse: /"
  POLY_B200_LIB=$L timeout 600 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 --nprobe 16 2>&1 | tail -1 | sed "s/^/$n np16: /"
  POLY_B200_LIB=$L timeout 900 python bench.py --config 4 --steps 10 --no-cpu-baseline --no-e2e > $O/cfg4_$n.json 2> $O/cfg4_$n.err; python -c "
import json
for l in open('$O/cfg4_$n.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$n cfg4 ms/step', d['ms_per_step'], 'codes/s', d['value'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_new.csv python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 1 > $O/ncu_new.log 2>&1
python tools/launches.py $O/launch_new.csv
