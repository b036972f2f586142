#!/bin/bash
# End-of-round evidence: GPU tests, smoke, every bench line, the headline launch list,
# a full ncu capture of the IVF top kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/fin_cfg1.json 2> gpurun_out/fin_cfg1.err; echo "cfg1 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --config 2 > gpurun_out/fin_cfg2.json 2> gpurun_out/fin_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config 4 > gpurun_out/fin_cfg4.json 2> gpurun_out/fin_cfg4.err; echo "cfg4 rc=$?"
timeout 900 python bench.py --config 3 --no-cpu-baseline > gpurun_out/fin_cfg3.json 2> gpurun_out/fin_cfg3.err; echo "cfg3 rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --per-ht 28,32 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches.csv $CMD > /dev/null 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on --profile-from-start off -k "regex:ivf_scan|residual_lut|coarse_refine" -c 4 \
    -o gpurun_out/fin_ivf_full python tools/prof_ivf.py --n 125000000 --nq 1024 --reps 1 --nprobe 16 > gpurun_out/fin_ivf_ncu.log 2>&1; echo "ivf ncu rc=$?"
for f in fin_cfg1 fin_ref fin_cfg2 fin_cfg4 fin_cfg3; do tail -1 gpurun_out/$f.json | cut -c1-300; done
