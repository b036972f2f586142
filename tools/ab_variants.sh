mkdir -p gpurun_out
for v in ${VARIANTS:-t12s4 t24s2}; do
  POLY_B200_LIB=tools/lib12/$v.so timeout 300 python bench.py --steps 10 --warmup 3 --per-ht 28,32 --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().splitlines()[-1]); print('$v', {k:round(v['ms_per_step'],2) for k,v in d['per_ht'].items()}, d['roofline']['kernel_ms_avg'])"
done
