#!/bin/bash
# Round evidence on HEAD: smoke, the GPU suite, every config's bench line, the reference arm, launch lists
# (gpurun -- bash tools/round_evidence.sh; the outputs are copied to profiles/ by hand)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/evidence
O=gpurun_out/evidence
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/cfg1.json 2> $O/cfg1.err; echo "cfg1 rc=$?"
timeout 900 python bench.py --impl reference > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launch_cfg1.csv python bench.py --steps 2 --warmup 1 --per-ht "" --no-cpu-baseline --no-e2e > $O/ncu1.log 2>&1; echo "ncu1=$?"
timeout 1500 python bench.py --config 2 --steps 5 > $O/cfg2.json 2> $O/cfg2.err; echo "cfg2 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_cfg2.csv env BENCH_PROFILE=1 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --per-nprobe "" > $O/ncu3.log 2>&1; echo "ncu3=$?"
timeout 600 python bench.py --config 0 > $O/cfg0.json 2> $O/cfg0.err; echo "cfg0 rc=$?"
timeout 1200 python bench.py --config 3 --steps 5 > $O/cfg3.json 2> $O/cfg3.err; echo "cfg3 rc=$?"
timeout 1500 python bench.py --config 4 --steps 10 --knn-full /tmp/knn_full.knng > $O/cfg4.json 2> $O/cfg4.err; echo "cfg4 rc=$?"
# launch lists of the other configs; the 8-rank by-list emulation (config 2, 1e9 codes, rank 0 measured on this GPU)
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_cfg4.csv env BENCH_PROFILE=1 python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu4.log 2>&1; echo "ncu4=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_cfg3.csv env BENCH_PROFILE=1 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --per-ht "" > $O/ncu3.log 2>&1; echo "ncu3=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launch_cfg0.csv env BENCH_PROFILE=1 python bench.py --config 0 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --per-ht "" > $O/ncu0.log 2>&1; echo "ncu0=$?"
timeout 2400 python tools/emulate_bylist.py > $O/emulate_bylist_rank0of8.json 2> $O/emulate.err; echo "emulate rc=$?"; tail -1 $O/emulate_bylist_rank0of8.json | cut -c1-600
