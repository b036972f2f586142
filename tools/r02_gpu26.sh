#!/bin/bash
# K6s round-1 seed: IVF parity, A/B (seed off / 1024 / 2048 rows) on the config-2 shape; flat parity (K2 knob cleanup)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ivf.py tests/test_gpu_survivors.py tests/test_gpu_parity.py -x -q > gpurun_out/t_seed.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t_seed.log
for v in "s0:-DPOLY_IVF_SEED_ROWS=0" "s1k:-DPOLY_IVF_SEED_ROWS=1024" "s2k:" "s4k:-DPOLY_IVF_SEED_ROWS=4096"; do
  n=${v%%:*}; f=${v#*:}
  bash tools/build_variant.sh $n $f > /dev/null 2>&1 || echo "build $n failed"
  POLY_B200_LIB=tools/lib12/$n.so timeout 600 python tools/prof_ivf.py --n 400000000 --nq 10000 --batch 10000 --reps 3 2>&1 | tail -1 | sed "s/^/$n: /"
done
