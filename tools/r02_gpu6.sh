#!/bin/bash
# K2t (role-split tensor-core flat scan): a quick smoke under a short timeout, parity suites, cfg1 bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python -c "
import numpy as np, oracle, paper_1609_01882_b200 as pb
z=np.load('tests/golden/golden_m8.npz'); p=np.load('tests/golden/pq_d128_m8.npz')
ix=pb.FlatIndex(pb.ProductQuantizer(8,8,128,p['codebooks'],p['perms'])); ix.add_codes(z['codes'])
ids,sc,cnt=ix.search_batch(z['queries'], pb.SearchParams(pb.Strategy.dual,100,24))
print('smoke ids equal:', np.array_equal(ids, z['dual24_ids']))
" > gpurun_out/k2t_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/k2t_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_survivors.py tests/test_gpu_sharded.py -x -q > gpurun_out/t_flat.log 2>&1; echo "flat tests rc=$?"; tail -8 gpurun_out/t_flat.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b_cfg1_k2t.json 2> gpurun_out/b_cfg1_k2t.err; echo "cfg1 rc=$?"; tail -c 300 gpurun_out/b_cfg1_k2t.err
