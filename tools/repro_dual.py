import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import load_pq
import paper_1609_01882_b200 as pb
pq8 = load_pq('pq_d128_m8.npz'); g = dict(np.load('tests/golden/golden_m8.npz'))
ix = pb.FlatIndex(pb.ProductQuantizer(8, 8, 128, pq8.codebooks, pq8.perms)); ix.add_codes(g['codes'])
for tau in [int(t) for t in sys.argv[1:]]:
    ids, sc, cnt = ix.search_batch(g['queries'], pb.SearchParams(pb.Strategy.dual, 100, tau))
    print(tau, np.array_equal(ids, g[f'dual{tau}_ids']), flush=True)
