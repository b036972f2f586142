# A/B of library variants at two database sizes (full N and a 1/8 shard), ht 24 only
mkdir -p gpurun_out
for v in $VARIANTS; do
  for n in 100000000 12500000; do
    POLY_B200_LIB=tools/lib12/$v.so timeout 300 python bench.py --n $n --per-ht "" --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/abs_${v}_$n.json 2>/dev/null
  done
  python -c "
import json
r=[]
for n in (100000000, 12500000):
    d=json.loads(open(f'gpurun_out/abs_${v}_{n}.json').read().splitlines()[-1]); r.append((n, round(d['ms_per_step'],3), round(d['roofline']['kernel_ms_avg'],3)))
print('$v', r)"
done
