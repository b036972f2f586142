import ctypes as C, sys, numpy as np, time
sys.path.insert(0, '.')
import oracle, paper_1609_01882_b200 as pb
from paper_1609_01882_b200._lib import lib
z = np.load('tests/golden/pq_d128_m8.npz')
pq = pb.ProductQuantizer(8, 8, 128, z['codebooks'], z['perms'])
seed = 160901882
centers = oracle.gen_centers(seed, 1000, 128)
ix = pb.FlatIndex(pq); ix.add_synthetic(seed, centers, 0, 1_000_000)
q = oracle.gen_points(seed, 3, 0, 256, centers)
for strat, tau in ((3, 32), (0, 0), (3, 64), (1, 0)):
    p = pb.SearchParams(pb.Strategy(strat), 100, tau)
    try:
        ix.search_batch(q, p); err = None
    except pb.PolyError as e:
        err = str(e)
    cc = np.empty(256, np.uint32); th = np.empty(256, np.uint64)
    lib.poly_b200_debug_counts(ix._h, cc.ctypes.data_as(C.c_void_p), th.ctypes.data_as(C.c_void_p), 256)
    print(strat, tau, 'err', err, 'ccount max/mean', cc.max(), cc.mean(), 'thr inf frac', (th == 2**64-1).mean(),
          'thr score', np.median((th >> 32).astype(np.uint32).view(np.float32)))
