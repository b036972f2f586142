"""Profiling driver: one dual search over a synthetic DB (use under ncu with
-k regex:scan_kernel; the main scan is the last scan_kernel launch of a batch)."""
import argparse, ctypes as C, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1609_01882_b200 as pb
from paper_1609_01882_b200 import synth
from paper_1609_01882_b200._lib import lib

ap = argparse.ArgumentParser()
ap.add_argument('--n', type=int, default=20_000_000)
ap.add_argument('--ht', type=int, default=32)
ap.add_argument('--nq', type=int, default=256)
ap.add_argument('--reps', type=int, default=1)
ap.add_argument('--m', type=int, default=8)
args = ap.parse_args()
dim = 16 * args.m
z = np.load('tests/golden/pq_d128_m8.npz' if args.m == 8 else 'tests/golden/pq_d256_m16.npz')
pq = pb.ProductQuantizer(args.m, 8, dim, z['codebooks'], z['perms'])
centers = synth.gen_centers(160901882, 1000 if args.m == 8 else 4096, dim)
ix = pb.FlatIndex(pq); ix.add_synthetic(160901882, centers, 0, args.n)
q = synth.gen_points(160901882, 3, 0, args.nq, centers)
p = pb.SearchParams(pb.Strategy.dual, 100, args.ht)
for r in range(args.reps):
    st = pb.SearchStats(); t = time.time()
    ix.search_batch(q, p, st)
    dt = time.time() - t
cc = np.empty(256, np.uint32); th = np.empty(256, np.uint64)
lib.poly_b200_debug_counts(ix._h, cc.ctypes.data_as(C.c_void_p), th.ctypes.data_as(C.c_void_p), 256)
print(f"n={args.n} ht={args.ht} {dt*1e3:.2f} ms  surv frac {st.survivors/(args.n*args.nq):.4f}  "
      f"cand max/mean {cc.max()}/{cc.mean():.0f}")
