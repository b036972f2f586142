#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
S="import numpy as np, paper_1609_01882_b200 as pb
z=np.load('tests/golden/golden_m8.npz'); p=np.load('tests/golden/pq_d128_m8.npz')
ix=pb.FlatIndex(pb.ProductQuantizer(8,8,128,p['codebooks'],p['perms'])); ix.add_codes(z['codes'])
for tau in (64, 24):
    ids,sc,cnt=ix.search_batch(z['queries'], pb.SearchParams(pb.Strategy.dual,100,tau))
    print(tau, 'ids equal:', np.array_equal(ids, z['dual%d_ids' % tau]))"
for v in "dbg1:-DPOLY_K2T_DEBUG=1" "stg4:-DPOLY_K2T_STG=4 -DPOLY_K2T_FQ=2" "fq2:-DPOLY_K2T_FQ=2" "base:"; do
  n=${v%%:*}; f=${v#*:}
  bash tools/build_variant.sh $n $f > /dev/null 2>&1 || echo "build $n failed"
  POLY_B200_LIB=tools/lib12/$n.so timeout 60 python -c "$S" > gpurun_out/k2tdbg_$n.log 2>&1; echo "$n rc=$?"; tail -2 gpurun_out/k2tdbg_$n.log
done
