#!/bin/bash
# HEAD validation after re-entry: full GPU suite; config-2 shape at 4e8 codes: round stats, launch list, round-1 chunk A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/g30
O=gpurun_out/g30
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -3 $O/pytest.log
timeout 900 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 --round-stats > $O/base.log 2>&1; tail -2 $O/base.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_4e8.csv python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/launches.py $O/launch_4e8.csv
for v in "c4k:-DPOLY_IVF_CHUNK=4096" "c2k:-DPOLY_IVF_CHUNK=2048"; do
  n=${v%%:*}; f=${v#*:}
  POLY_B200_LIB=tools/lib12/$n.so timeout 600 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 2>&1 | tail -1 | sed "s/^/$n: /"
done
