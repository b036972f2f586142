#!/bin/bash
# K3 staging A/B (k <= 512: 4096 vs 6144 vs 8192 staged keys) on the config-2 shape (4e8, 10,000 queries) and config 1
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "tk4:" "tk6:-DPOLY_TK_SMALLK_KEYS=6144" "tk8:-DPOLY_TK_SMALLK_KEYS=8192"; do
  n=${v%%:*}; f=${v#*:}
  bash tools/build_variant.sh $n $f > /dev/null 2>&1 || echo "build $n failed"
  POLY_B200_LIB=tools/lib12/$n.so timeout 600 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 2>&1 | tail -1 | sed "s/^/$n: /"
  POLY_B200_LIB=tools/lib12/$n.so timeout 300 python bench.py --steps 5 --warmup 2 --per-ht "" --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$n cfg1', round(d['ms_per_step'],3))"
done
