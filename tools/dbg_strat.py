import sys, numpy as np
sys.path.insert(0, '.')
import paper_1609_01882_b200 as pb
z = np.load('tests/golden/pq_d128_m8.npz'); g = np.load('tests/golden/golden_m8.npz')
pq = pb.ProductQuantizer(8, 8, 128, z['codebooks'], z['perms'])
for strat in sys.argv[1:]:
    ix = pb.FlatIndex(pq); ix.add_codes(g['codes'])
    try:
        ids, sc, cnt = ix.search_batch(g['queries'], pb.SearchParams(pb.strategy_from_string(strat), 100, 24))
        print(strat, 'ok', (ids == g[f'{strat}_ids'] if strat != 'dual' else ids[:1,:3]).all() if strat!='dual' else ids[0,:3])
    except Exception as e:
        print(strat, 'ERR', e); break
