#!/bin/bash
# Round evidence: GPU tests, bench lines of every config, IVF launch lists.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_all.log
timeout 600 python bench.py > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "cfg1 rc=$?"
timeout 900 python bench.py --config 2 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config 4 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 rc=$?"
for np in 16 64; do
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/ivf_cfg2_b1024_np${np}_launches.csv \
      python tools/prof_ivf.py --n 125000000 --nq 1024 --reps 1 --nprobe $np > /dev/null 2>&1
done
python tools/launches.py gpurun_out/ivf_cfg2_b1024_np*_launches.csv
for c in 1 2 4 3; do tail -1 gpurun_out/bench_cfg$c.json | cut -c1-400; done
