#!/bin/bash
# IVF evidence: cfg2 / cfg4 bench lines, 1024-query launch lists, full ncu of the IVF kernels.
mkdir -p gpurun_out
timeout 900 python bench.py --config 2 > gpurun_out/fin_cfg2.json 2> gpurun_out/fin_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config 4 > gpurun_out/fin_cfg4.json 2> gpurun_out/fin_cfg4.err; echo "cfg4 rc=$?"
for np in 16 64; do
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/ivf_cfg2_b2048_np${np}_launches.csv \
      python tools/prof_ivf.py --n 125000000 --nq 2048 --reps 1 --nprobe $np > /dev/null 2>&1
done
BENCH_PROFILE=1 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/cfg4_launches.csv python bench.py --config 4 --steps 1 --warmup 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k "regex:ivf_scan|residual_lut|coarse_refine|topk" -c 7 \
    -o gpurun_out/fin_ivf_full python tools/prof_ivf.py --n 125000000 --nq 2048 --reps 1 --nprobe 16 > gpurun_out/fin_ivf_ncu.log 2>&1; echo "ivf ncu rc=$?"
python tools/launches.py gpurun_out/ivf_cfg2_b2048_np*_launches.csv gpurun_out/cfg4_launches.csv
