"""Coarse quantization alone (K5t + K5q), for ncu: nlist 65,536 cells (BASELINE cfg2),
2048 queries per call, nprobe 16.  python tools/prof_coarse.py [--nlist N] [--dim D] [--reps R]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1609_01882_b200 as pb  # noqa: E402
from paper_1609_01882_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nlist", type=int, default=65536)
ap.add_argument("--dim", type=int, default=128)
ap.add_argument("--nq", type=int, default=2048)
ap.add_argument("--nprobe", type=int, default=16)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
SEED = 160901882
m = a.dim // 16
z = np.load(os.path.join(ROOT, "tests", "golden", "pq_d128_m8.npz" if m == 8 else "pq_d256_m16.npz"))
pq = pb.ProductQuantizer(m, 8, a.dim, z["codebooks"], z["perms"])
centers = synth.gen_centers(SEED, 1000 if m == 8 else 4096, a.dim)
coarse = synth.gen_points(SEED, 1, 0, a.nlist, centers)
ivf = pb.IVFIndex(pq, coarse)
dq = torch.empty((a.nq, a.dim), dtype=torch.float32, device="cuda")
pb.gen_points_device(centers, SEED, 3, 0, a.nq, dq)
out = torch.empty((a.nq, a.nprobe), dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    ivf.probe_keys_device(dq, a.nprobe, out, stream=s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    ivf.probe_keys_device(dq, a.nprobe, out, stream=s)
e1.record()
torch.cuda.synchronize()
print(f"coarse quantization: {e0.elapsed_time(e1) / a.reps * 1e3:.1f} us per {a.nq} queries (nlist {a.nlist}, dim {a.dim})")
