#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 compute-sanitizer --tool memcheck --print-limit 20 python -c "
import numpy as np, paper_1609_01882_b200 as pb
z=np.load('tests/golden/golden_m8.npz'); p=np.load('tests/golden/pq_d128_m8.npz')
ix=pb.FlatIndex(pb.ProductQuantizer(8,8,128,p['codebooks'],p['perms'])); ix.add_codes(z['codes'])
ids,sc,cnt=ix.search_batch(z['queries'], pb.SearchParams(pb.Strategy.dual,100,24))
print('smoke ids equal:', np.array_equal(ids, z['dual24_ids']))
" > gpurun_out/k2t_san.log 2>&1; echo "san rc=$?"; grep -v "^=========     at\|^=========         " gpurun_out/k2t_san.log | head -40
