#!/bin/bash
# K2t variants (filter quads) vs K2 (POLY_K2T=0) on config 1, ht 24 / 28
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "k2:-DPOLY_K2T=0" "fq2:-DPOLY_K2T_FQ=2" "fq1:-DPOLY_K2T_FQ=1"; do
  n=${v%%:*}; f=${v#*:}
  bash tools/build_variant.sh $n $f > /dev/null 2>&1 || echo "build $n failed"
  POLY_B200_LIB=tools/lib12/$n.so timeout 300 python bench.py --steps 5 --warmup 2 --per-ht 28 --no-cpu-baseline --no-e2e > gpurun_out/k2tab_$n.json 2> gpurun_out/k2tab_$n.err
  python -c "
import json; d=json.loads(open('gpurun_out/k2tab_$n.json').read().splitlines()[-1]); print('$n', {k:round(v['ms_per_step'],2) for k,v in d['per_ht'].items()})" || tail -3 gpurun_out/k2tab_$n.err
done
