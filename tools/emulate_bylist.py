"""Per-rank cost of by-list IVF sharding at W ranks, measured on one GPU (config 2).

The pool has one B200 per box, so the 8-rank run cannot be timed directly.  This builds
the full config-2 index (N codes) and rank R's by-list shard of the same data
(assign_lists over the list sizes, bench.build_ivf_by_list), then times with CUDA events
what rank R does per 10,000-query step under the two-phase protocol:

  coarse     enumerate_cells for its 1/W slice of the queries (probe_keys_device)
  phase 1    round 1 over the first probes it owns
  phase 2    round 2 over its other probed lists under the global bound -- the bound the
             min-reduce would deliver is exactly the owner's round-1 k-th key, i.e. the
             full index's own phase-1 output, which is what is passed in
  merge      K3 over W x k keys per query (merge_keys_device, parts = W)

and adds the collectives at stated NVLink rates.  The 1-GPU step is the full index's
device search of the same queries.  Prints one JSON line.

    python tools/emulate_bylist.py [--n 1e9] [--world 8] [--rank 0] [--nprobe 16]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1609_01882_b200 as pb  # noqa: E402
from paper_1609_01882_b200 import synth  # noqa: E402
from paper_1609_01882_b200.distributed import shard_range  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e9)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--nprobe", type=int, default=16)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--nvlink-gbs", type=float, default=350.0, help="all-gather / all-reduce bus bandwidth assumed")
a = ap.parse_args()

args = argparse.Namespace(config=2, c=bench.CONFIGS[2], n=int(a.n), coarse="sample")
c = args.c
k, nq, W, R = 100, c["nq"], a.world, a.rank
centers = synth.gen_centers(bench.SEED, c["ncent"], c["dim"])
coarse = bench.make_coarse(args, pb, synth, centers, False)
t0 = time.time()
full, _ = bench.build_ivf(args, pb, torch, 0, 0, args.n, coarse, centers, False)
shard, _ = bench.build_ivf_by_list(args, pb, torch, 0, R, W, coarse, centers, False)
setup = time.time() - t0
for ix in (full, shard):
    ix.set_batch(nq)
dq = torch.empty((nq, c["dim"]), dtype=torch.float32, device="cuda")
pb.gen_points_device(centers, bench.SEED, 3, 0, nq, dq)
p = pb.CoarseParams(pb.Strategy.dual, k, c["ht"], a.nprobe, 0)
s = torch.cuda.current_stream()
sp = s.cuda_stream


def timed(fn, reps=a.reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


o = (torch.empty((nq, k), dtype=torch.int64, device="cuda"), torch.empty((nq, k), dtype=torch.float32, device="cuda"),
     torch.empty(nq, dtype=torch.int32, device="cuda"))
t_full = timed(lambda: full.search_device(dq, p, o[0], o[1], o[2], sp))
st_full = pb.SearchStats()
full.search_device(dq, p, o[0], o[1], o[2], sp, st_full)

probes = torch.empty((nq, a.nprobe), dtype=torch.int64, device="cuda")
full.probe_keys_device(dq, a.nprobe, probes, stream=sp)
b0, b1 = shard_range(nq, W, R)
sl = torch.empty((b1 - b0, a.nprobe), dtype=torch.int64, device="cuda")
t_coarse = timed(lambda: full.probe_keys_device(dq[b0:b1], a.nprobe, sl, stream=sp))

thr_g = torch.empty(nq, dtype=torch.int64, device="cuda")  # the global bound = the owner's round-1 k-th key
tk = torch.empty((nq, k), dtype=torch.int64, device="cuda")
tc = torch.empty(nq, dtype=torch.int32, device="cuda")
full.search_keys_phase_device(dq, p, probes, 1, thr_g, stream=sp)
full.search_keys_phase_device(dq, p, probes, 2, thr_g.clone(), tk, tc, stream=sp)
thr_l = torch.empty(nq, dtype=torch.int64, device="cuda")
keys = torch.empty((W, nq, k), dtype=torch.int64, device="cuda")
cnts = torch.empty((W, nq), dtype=torch.int32, device="cuda")
st_r = pb.SearchStats()


def rank_step():
    shard.search_keys_phase_device(dq, p, probes, 1, thr_l, stream=sp)
    shard.search_keys_phase_device(dq, p, probes, 2, thr_g.clone(), keys[0], cnts[0], stream=sp)


t_rank = timed(rank_step)
shard.search_keys_phase_device(dq, p, probes, 1, thr_l, stream=sp)
shard.search_keys_phase_device(dq, p, probes, 2, thr_g.clone(), keys[0], cnts[0], stream=sp, stats=st_r)
for r in range(1, W):  # stand-in parts for the merge's cost (same sizes)
    keys[r].copy_(keys[0])
    cnts[r].copy_(cnts[0])
t_merge = timed(lambda: full.merge_keys_device(keys, cnts, W, nq, k, o[0], o[1], o[2], stream=sp))
per = (nq + W - 1) // W  # all-to-all exchange: this rank merges its query slice only
ks = keys[:, :per].contiguous()
cs = cnts[:, :per].contiguous()
t_merge_slice = timed(lambda: full.merge_keys_device(ks, cs, W, per, k, o[0], o[1], o[2], stream=sp))
# collectives per step: probe keys all-gather (nq x nprobe x 8 B), bound all-reduce (nq x 8 B),
# key + count all-gather (W x nq x (k x 8 + 4) B received per rank)
bw = a.nvlink_gbs * 1e9
comm = {"probe_allgather_ms": nq * a.nprobe * 8 / bw * 1e3, "bound_allreduce_ms": 2 * nq * 8 / bw * 1e3,
        "key_allgather_ms": W * nq * (k * 8 + 4) / bw * 1e3, "latency_ms": 3 * 0.02}
t_comm = sum(comm.values())
per_rank = t_coarse + t_rank + t_merge + t_comm
# all-to-all exchange (ShardedSearch(exchange="alltoall"), the bench's IVF default): keys of the
# other slices out, this slice's keys in, merged slices all-gathered
comm_a2a = {"probe_allgather_ms": comm["probe_allgather_ms"], "bound_allreduce_ms": comm["bound_allreduce_ms"],
            "key_alltoall_ms": (W - 1) / W * nq * (k * 8 + 4) / bw * 1e3,
            "result_allgather_ms": (W - 1) / W * nq * (k * 12 + 4) / bw * 1e3, "latency_ms": 4 * 0.02}
per_rank_a2a = t_coarse + t_rank + t_merge_slice + sum(comm_a2a.values())
sizes = np.diff(shard.list_offsets().astype(np.int64))
print(json.dumps({
    "what": f"by-list sharding, rank {R} of {W}, config 2: N={args.n} codes, nq={nq} per step, nprobe={a.nprobe}",
    "one_gpu_step_ms": t_full, "one_gpu_scanned": st_full.scanned,
    "rank": {"coarse_slice_ms": t_coarse, "phase1_plus_phase2_ms": t_rank, "merge_ms": t_merge,
             "scanned": st_r.scanned, "codes_held": int(sizes.sum())},
    "collectives_est": {k2: round(v, 4) for k2, v in comm.items()},
    "allgather": {"per_rank_step_ms": per_rank, "projected_speedup": t_full / per_rank,
                  "projected_efficiency": t_full / per_rank / W},
    "alltoall": {"merge_slice_ms": t_merge_slice, "collectives_est": {k2: round(v, 4) for k2, v in comm_a2a.items()},
                 "per_rank_step_ms": per_rank_a2a, "projected_speedup": t_full / per_rank_a2a,
                 "projected_efficiency": t_full / per_rank_a2a / W},
    "setup_s": round(setup, 1)}), flush=True)
