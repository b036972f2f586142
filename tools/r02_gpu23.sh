#!/bin/bash
# K6 A/B: register prefetch of the next block x CTAs per SM, config-2 shape at 4e8 codes, 10,000 queries
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "base:" "pf12:-DPOLY_K6_PREFETCH=1" "pf10:-DPOLY_K6_PREFETCH=1 -DPOLY_K6_MINB=10" "pf8:-DPOLY_K6_PREFETCH=1 -DPOLY_K6_MINB=8" "b10:-DPOLY_K6_MINB=10"; do
  n=${v%%:*}; f=${v#*:}
  bash tools/build_variant.sh $n $f > /dev/null 2>&1 || echo "build $n failed"
  grep -A2 "ivf_list_scan_kernelILi8ELi3ELb0" tools/lib12/$n/*.log 2>/dev/null | head -0
  POLY_B200_LIB=tools/lib12/$n.so timeout 600 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 2>&1 | tail -1 | sed "s/^/$n: /"
done
