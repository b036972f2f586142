#!/bin/bash
# A/B of IVF library variants on config 2 (bench --config 2): VARIANTS="name:batch ..."
mkdir -p gpurun_out
for vb in ${VARIANTS:-nqb256:256}; do
  v=${vb%%:*}; b=${vb##*:}
  POLY_B200_LIB=tools/lib12/$v.so timeout 600 python bench.py --config 2 --steps ${STEPS:-10} --warmup 3 --ivf-batch $b ${EXTRA} > gpurun_out/abivf_$v.json 2> gpurun_out/abivf_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/abivf_$v.json').read().splitlines()[-1]); print('$v b=$b', {k:(round(v['ms_per_step'],3), '%.3e'%v['value'], round(v['survivor_frac'],3)) for k,v in d['per_nprobe'].items()})" || tail -5 gpurun_out/abivf_$v.err
done
