#!/usr/bin/env python
"""Polysemous dual search on B200 -- the BASELINE.json headline metric.

Workload (BASELINE.json configs[1], "cfg1"): flat polysemous PQ, d = 128
mixture, m = 8 x 8-bit codes (64-bit), N = 100,000,000 codes (800 MB) sharded
over the ranks, nq = 10,000 queries in batches of 256, k = 100, headline
ht = 24 (the Table 1 calibration rule: tau filters >= ~94% of the codes);
ht = 28 and 32 are reported under "per_ht".  Data are synthetic (the seeded
mixture of BASELINE.json).

One step = one 256-query batch through the whole path: K1 LUT + query code,
K0 warm-up + K2 fused filter/ADC/candidate scan, K3 exact top-k, key -> id;
at N > 1 plus the NCCL all-gather of per-shard top-k keys and the K3 merge.
`value` = codes scanned per second over the whole job (256 * N_total per
step), queries and codes resident in HBM; `e2e` = the same with the queries
copied from pinned host memory and the results (ids, scores, counts,
survivors) copied back inside the timed region.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DB codes scanned/sec (filter+ADC+top-k)"
UNIT = "codes/s"
SEED = 160901882
BATCH = 256
IVF_BATCH = 2048  # configs 2/4 (BASELINE.json names no batch size there): the library's IVF batch
NQ = 10_000
# BASELINE.json configs: 1 = flat 64-bit codes (headline), 3 = wide 128-bit codes
CONFIGS = {
    1: dict(dim=128, ncent=1000, m=8, n=100_000_000, ht=24, per_ht="28,32", pq="pq_d128_m8.npz"),
    3: dict(dim=256, ncent=4096, m=16, n=200_000_000, ht=56, per_ht="48,64", pq="pq_d256_m16.npz"),
    # IVF: the per-GPU share of the 1B-code config (1e9 / 8 GPUs)
    2: dict(dim=128, ncent=1000, m=8, n=125_000_000, ht=26, per_ht="", pq="pq_ivf65536_d128_m8.npz",
            nlist=65536, nprobe=16, per_nprobe="64"),
    # approximate k-NN graph: every database vector queries the rest
    4: dict(dim=256, ncent=4096, m=16, n=10_000_000, ht=52, per_ht="", pq="pq_ivf16384_d256_m16.npz",
            nlist=16384, nprobe=32, per_nprobe="", knn_k=10),
}
NCENT = 1000
DIM = 128
M = 8
PQFILE = "pq_d128_m8.npz"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=None, help="total database codes (default: the config's N)")
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--ht", type=int, default=None)
    ap.add_argument("--per-ht", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-queries", type=int, default=256, help="queries in the CPU-baseline sample")
    ap.add_argument("--ivf-batch", type=int, default=IVF_BATCH, help="queries per step for configs 2 and 4")
    ap.add_argument("--ref-n", type=int, default=8_000_000, help="codes in the --impl reference sample")
    args = ap.parse_args()
    global NCENT, DIM, M, PQFILE
    c = CONFIGS[args.config]
    NCENT, DIM, M, PQFILE = c["ncent"], c["dim"], c["m"], c["pq"]
    args.n = c["n"] if args.n is None else args.n
    args.ht = c["ht"] if args.ht is None else args.ht
    args.per_ht = c["per_ht"] if args.per_ht is None else args.per_ht
    if args.config in (2, 4) and args.impl == "reference":
        raise SystemExit("--impl reference is defined for the flat configs (1, 3)")
    return args


def config(args, world):
    return {
        "workload": f"cfg{args.config} flat polysemous: N={args.n} {8 * M}-bit codes (m={M}, nbits=8, d={DIM} "
                    f"mixture of {NCENT}), nq={NQ} in batches of {BATCH}, k={args.k}, ht={args.ht}",
        "n_codes": args.n, "m": M, "nbits": 8, "dim": DIM, "k": args.k, "ht": args.ht, "batch": BATCH, "nq": NQ,
        "strategy": "dual", "parallelism": f"db-shard{world}",
        "l2": f"inputs larger than L2 ({args.n * M / 1e6:.0f} MB of codes vs 126 MB L2); no flush needed",
    }


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.path = tempfile.mktemp(suffix=".csv")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-i", ",".join(str(g) for g in gpus), "-lms", "100"],
                                      stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank):
    """The reference's own CPU search (oracle/_ref: reference sources compiled in
    place; FlatIndex::search restated per SPEC from its primitives) on the host."""
    if rank != 0:
        return
    import oracle
    from paper_1609_01882_b200 import synth
    threads = os.cpu_count()
    z = np.load(os.path.join(ROOT, "tests", "golden", PQFILE))
    pq = oracle.PQ(M, 8, DIM, z["codebooks"], z["perms"])
    kind = "reference" if oracle.ref_available() else "port"
    centers = synth.gen_centers(SEED, NCENT, DIM)
    t = time.time()
    codes = np.empty((args.ref_n, M), np.uint8)
    step = 1 << 20
    for r0 in range(0, args.ref_n, step):
        x = oracle.gen_points(SEED, 2, r0, min(step, args.ref_n - r0), centers)
        codes[r0:r0 + len(x)] = oracle.ref_encode_batch(pq, x, threads) if kind == "reference" else oracle.encode(pq, x, threads)
    setup = time.time() - t
    queries = synth.gen_points(SEED, 3, 0, NQ, centers)

    def step_fn(i):
        q = queries[(i * BATCH) % (NQ - NQ % BATCH):][:BATCH]
        if kind == "reference":
            oracle.ref_search(pq, codes, q, args.k, tau=args.ht, threads=threads)
        else:
            oracle.search(pq, codes, q, args.k, tau=args.ht, threads=threads)

    for i in range(args.warmup):
        step_fn(i)
    t = time.perf_counter()
    for i in range(args.steps):
        step_fn(args.warmup + i)
    dt = time.perf_counter() - t
    value = args.steps * BATCH * args.ref_n / dt
    sample = (f"each step: {BATCH} queries x {args.ref_n} codes of the cfg1 mixture (encoded by the reference's "
              f"encode_batch), two-pass dual search, ht={args.ht}, k={args.k}; {threads} threads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8/f32", "data": "synthetic",
            "config": config(args, args.gpus), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": round(setup, 1)}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ IVF (configs 2 and 4)
def run_ivf(args, rank, world, local):
    """search_coarse throughput: codes scanned/s over the probed lists (config 2),
    or the k-NN graph where every stored vector is a query (config 4)."""
    import torch
    import paper_1609_01882_b200 as pb
    from paper_1609_01882_b200 import synth
    from paper_1609_01882_b200.distributed import shard_range
    c = CONFIGS[args.config]
    knn = args.config == 4
    norm = knn
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    z = np.load(os.path.join(ROOT, "tests", "golden", PQFILE))
    pq = pb.ProductQuantizer(M, 8, DIM, z["codebooks"], z["perms"])
    centers = synth.gen_centers(SEED, NCENT, DIM)
    coarse = synth.gen_points(SEED, 1, 0, c["nlist"], centers, normalize=norm)  # the fixture's coarse recipe
    ivf = pb.IVFIndex(pq, coarse, device=local)
    row0, row1 = shard_range(args.n, world, rank)
    # build (setup, untimed): GPU generator, TF32-GEMM nearest-cell assignment,
    # exact residual encoding through the C ABI
    t = time.time()
    torch.backends.cuda.matmul.allow_tf32 = True
    dc = torch.from_numpy(coarse).cuda()
    cn = (dc * dc).sum(1)
    chunk = 1 << 20
    xbuf = torch.empty((chunk, DIM), dtype=torch.float32, device="cuda")
    cells = torch.empty(chunk, dtype=torch.int32, device="cuda")
    for r in range(row0, row1, chunk):
        nb = min(chunk, row1 - r)
        x = xbuf[:nb]
        pb.gen_points_device(centers, SEED, 2, r, nb, x, device=local, normalize=norm)
        for b in range(0, nb, 8192):
            xs = x[b:b + 8192]
            cells[b:b + xs.shape[0]] = torch.argmin(cn[None, :] - 2.0 * (xs @ dc.T), dim=1).to(torch.int32)
        ivf.add_device(x, cells[:nb], r)
    torch.cuda.synchronize()
    setup_s = time.time() - t
    if knn:
        try:
            return run_knn(args, c, ivf, centers, setup_s, rank, world, local, row0, row1)
        finally:
            if dist is not None:
                dist.destroy_process_group()
    dq = torch.empty((NQ, DIM), dtype=torch.float32, device="cuda")
    pb.gen_points_device(centers, SEED, 3, 0, NQ, dq, device=local)
    stream = torch.cuda.current_stream()
    k = args.k
    B = args.ivf_batch
    o_ids = torch.empty((B, k), dtype=torch.int64, device="cuda")
    o_sc = torch.empty((B, k), dtype=torch.float32, device="cuda")
    o_cnt = torch.empty(B, dtype=torch.int32, device="cuda")
    nbatches = NQ // B
    results = {}
    if dist is not None:
        # every cell's list holds this rank's id range; per-rank top-k
        # keys are all-gathered over NCCL and merged exactly (IVFIndexEngine + ShardedSearch)
        from paper_1609_01882_b200.distributed import IVFIndexEngine, ShardedSearch
        engine = IVFIndexEngine(ivf, split_coarse=True)  # coarse quantization split by query
        sharded = ShardedSearch(engine)

    def step(i, p, st=None):
        q = dq[(i % nbatches) * B:][:B]
        if dist is None:
            ivf.search_device(q, p, o_ids, o_sc, o_cnt, stream.cuda_stream, st)
        else:
            engine.stats = st
            sharded.search_batch(q, p, (o_ids, o_sc, o_cnt))

    for nprobe in [c["nprobe"]] + [int(x) for x in c["per_nprobe"].split(",") if x]:
        p = pb.CoarseParams(pb.Strategy.dual, k, args.ht, nprobe, 0)
        steps = args.steps if nprobe == c["nprobe"] else max(3, args.steps // 2)
        scanned = surv = 0
        for i in range(args.warmup, args.warmup + steps):  # per-batch work (untimed)
            st = pb.SearchStats()
            step(i, p, st)
            scanned += st.scanned
            surv += st.survivors
        if dist is not None:  # codes scanned by all ranks
            t = torch.tensor([scanned, surv], dtype=torch.float64, device="cuda")
            dist.all_reduce(t)
            scanned, surv = int(t[0].item()), int(t[1].item())
        for i in range(args.warmup):
            step(i, p)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        l0 = pb.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.warmup, args.warmup + steps):
            step(i, p)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if dist is not None:  # max over ranks
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        results[nprobe] = {"value": scanned / (ms / 1e3), "ms_per_step": ms / steps,
                           "scanned_per_query": scanned / (steps * B), "survivor_frac": surv / max(scanned, 1),
                           "gpu_launches": pb.launch_count() - l0, "steps": steps}
    head = results[c["nprobe"]]
    line = {"metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": head["steps"],
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8/f32", "data": "synthetic (seeded Gaussian mixture, BASELINE cfg2)",
            "config": {"workload": f"cfg2 IVF+polysemous: nlist={c['nlist']}, N={args.n} codes over {world} GPU(s) (the "
                                   f"per-GPU share of 1e9 over 8 at N=1), PQ m={M} on residuals, nq={NQ} in batches of "
                                   f"{B}, nprobe={c['nprobe']}, k={k}, ht={args.ht}",
                       "nlist": c["nlist"], "n_codes": args.n, "m": M, "nprobe": c["nprobe"], "k": k, "ht": args.ht,
                       "parallelism": f"db-shard{world} (ids within every list) + query-split coarse quantization + NCCL probe / key all-gathers",
                       "coarse": "training-stream rows [0, nlist) (sampled coarse quantizer; DESIGN.md)",
                       "build_assignment": "TF32 GEMM argmin (setup only)"},
            "gpu_launches": head["gpu_launches"], "per_nprobe": {str(kk): v for kk, v in results.items()},
            "setup_s": round(setup_s, 1)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_knn(args, c, ivf, centers, setup_s, rank, world, local, row0, row1):
    """Config 4: the k-NN graph.  A step = 256 stored vectors searched against the
    whole index with k + 1 neighbours and the self-match removed."""
    import torch
    import paper_1609_01882_b200 as pb
    k = c["knn_k"]
    p = pb.CoarseParams(pb.Strategy.dual, k, args.ht, c["nprobe"], 0)
    stream = torch.cuda.current_stream()
    steps = args.steps
    B = args.ivf_batch
    nrows = (args.warmup + steps) * B
    dx = torch.empty((nrows, DIM), dtype=torch.float32, device="cuda")
    pb.gen_points_device(centers, SEED, 2, row0, nrows, dx, device=local, normalize=True)
    o_ids = torch.empty((B, k), dtype=torch.int64, device="cuda")
    o_sc = torch.empty((B, k), dtype=torch.float32, device="cuda")
    o_cnt = torch.empty(B, dtype=torch.int32, device="cuda")
    scanned = 0
    p1 = pb.CoarseParams(pb.Strategy.dual, k + 1, args.ht, c["nprobe"], 0)
    for i in range(args.warmup, args.warmup + steps):  # per-batch work (untimed)
        st = pb.SearchStats()
        qb = dx[i * B:(i + 1) * B]
        ob = (torch.empty((B, k + 1), dtype=torch.int64, device="cuda"),
              torch.empty((B, k + 1), dtype=torch.float32, device="cuda"))
        ivf.search_device(qb, p1, ob[0], ob[1], None, stream.cuda_stream, st)
        scanned += st.scanned
    for i in range(args.warmup):
        ivf.knn_graph_device(dx[i * B:(i + 1) * B], row0 + i * B, p, o_ids, o_sc, o_cnt,
                             stream.cuda_stream)
    torch.cuda.synchronize()
    l0 = pb.launch_count()
    prof = os.environ.get("BENCH_PROFILE") == "1"  # ncu --profile-from-start off: the timed steps only
    if prof:
        torch.cuda.profiler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.warmup, args.warmup + steps):
        ivf.knn_graph_device(dx[i * B:(i + 1) * B], row0 + i * B, p, o_ids, o_sc, o_cnt,
                             stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if prof:
        torch.cuda.profiler.stop()
    ms = e0.elapsed_time(e1)
    rows = row1 - row0
    line = {"metric": METRIC, "value": scanned / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8/f32", "data": "synthetic (unit-normalised mixture, BASELINE cfg4)",
            "config": {"workload": f"cfg4 k-NN graph: N={args.n} d={DIM} unit-normalised, IVF {c['nlist']} + PQ "
                                   f"m={M}, every vector queries the rest, nprobe={c['nprobe']}, ht={args.ht}, k={k}",
                       "n_codes": args.n, "nlist": c["nlist"], "m": M, "nprobe": c["nprobe"], "k": k,
                       "ht": args.ht, "queries_per_step": B},
            "scanned_per_query": scanned / (steps * B),
            "graph_time_est_s": rows / B * ms / steps / 1e3, "gpu_launches": pb.launch_count() - l0,
            "setup_s": round(setup_s, 1)}
    if rank == 0:
        print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def cpu_baseline(args, index, dq_host):
    """Reference CPU search (oracle/_ref) on one full step of the workload:
    256 queries over all N codes, every host thread."""
    import oracle
    z = np.load(os.path.join(ROOT, "tests", "golden", PQFILE))
    pq = oracle.PQ(M, 8, DIM, z["codebooks"], z["perms"])
    codes = index.codes()
    q = dq_host[:args.cpu_queries]
    threads = os.cpu_count()
    kind = "reference" if oracle.ref_available() else "port"
    t = time.perf_counter()
    if kind == "reference":
        oracle.ref_search(pq, codes, q, args.k, tau=args.ht, threads=threads)
    else:
        oracle.search(pq, codes, q, args.k, tau=args.ht, threads=threads)
    dt = time.perf_counter() - t
    return {"value": len(q) * codes.shape[0] / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{len(q)} queries x all {codes.shape[0]} codes (one full step), two-pass dual ht={args.ht}, "
                      f"k={args.k}, {dt:.1f} s"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if args.config in (2, 4):
        run_ivf(args, rank, world, local)
        return

    import torch
    import paper_1609_01882_b200 as pb
    from paper_1609_01882_b200 import synth

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    z = np.load(os.path.join(ROOT, "tests", "golden", PQFILE))
    pq = pb.ProductQuantizer(M, 8, DIM, z["codebooks"], z["perms"])
    centers = synth.gen_centers(SEED, NCENT, DIM)
    from paper_1609_01882_b200.distributed import shard_range
    row0, row1 = shard_range(args.n, world, rank)
    nloc = row1 - row0
    t = time.time()
    index = pb.FlatIndex(pq, device=local)
    index.add_synthetic(SEED, centers, row0, nloc)   # GPU generator + encoder, ids = global rows
    setup_s = time.time() - t

    dq = torch.empty((NQ, DIM), dtype=torch.float32, device="cuda")
    pb.gen_points_device(centers, SEED, 3, 0, NQ, dq, device=local)
    hq = dq.cpu().pin_memory()
    nbatches = NQ // BATCH
    k = args.k
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    o_ids = torch.empty((BATCH, k), dtype=torch.int64, device="cuda")
    o_sc = torch.empty((BATCH, k), dtype=torch.float32, device="cuda")
    o_cnt = torch.empty(BATCH, dtype=torch.int32, device="cuda")
    o_surv = torch.empty(BATCH, dtype=torch.int64, device="cuda")
    if world > 1:
        from paper_1609_01882_b200.distributed import FlatIndexEngine, ShardedSearch
        sharded = ShardedSearch(FlatIndexEngine(index), device="cuda")

    def step(i, ht, q=None):
        qb = dq[(i % nbatches) * BATCH:][:BATCH] if q is None else q
        p = pb.SearchParams(pb.Strategy.dual, k, ht)
        if world == 1:
            index.search_batch_device(qb, p, o_ids, o_sc, o_cnt, None, stream=sptr)
        else:  # local shard scan, NCCL all-gather of top-k keys, K3 merge
            sharded.search_batch(qb, p, out=(o_ids, o_sc, o_cnt))

    def timed(ht, steps, warmup, profile=False):
        for i in range(warmup):
            step(i, ht)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            index.profile_enable(True)
        surv = 0
        l0 = pb.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            step(warmup + i, ht)
        e1.record(stream)
        torch.cuda.synchronize()
        launches = pb.launch_count() - l0
        ms = e0.elapsed_time(e1)
        scan = index.profile_read() if profile else None
        if profile:
            index.profile_enable(False)
        # survivor fraction of one batch on this shard (outside the timed region)
        st = pb.SearchStats()
        index.search_batch_device(dq[:BATCH], pb.SearchParams(pb.Strategy.dual, k, ht), o_ids, o_sc, o_cnt, None,
                                  stream=sptr, stats=st)
        surv = st.survivors
        if dist:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, launches, scan, surv

    # ---- headline (device-resident)
    clocks = ClockSampler([local] if world == 1 else list(range(world))) if rank == 0 else None
    ms, launches, scan, surv_last = timed(args.ht, args.steps, args.warmup, profile=True)
    clk = clocks.stop() if clocks else None
    value = args.steps * BATCH * args.n / (ms / 1e3)

    # ---- e2e: pinned host queries in, results out, inside the timed region
    h_ids = torch.empty((BATCH, k), dtype=torch.int64).pin_memory()
    h_sc = torch.empty((BATCH, k), dtype=torch.float32).pin_memory()
    h_cnt = torch.empty(BATCH, dtype=torch.int32).pin_memory()
    qdev = torch.empty((BATCH, DIM), dtype=torch.float32, device="cuda")

    def e2e_step(i):
        qdev.copy_(hq[(i % nbatches) * BATCH:][:BATCH], non_blocking=True)
        step(i, args.ht, q=qdev)
        if rank == 0:
            h_ids.copy_(o_ids, non_blocking=True)
            h_sc.copy_(o_sc, non_blocking=True)
            h_cnt.copy_(o_cnt, non_blocking=True)

    for i in range(args.warmup):
        e2e_step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        e2e_step(args.warmup + i)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": args.steps * BATCH * args.n / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": BATCH * DIM * 4,
           "d2h_bytes_per_step": (BATCH * k * 12 + BATCH * 4) if rank == 0 else 0,
           "ms_per_step": e2e_ms / args.steps}

    # ---- per-ht sweep (device-resident)
    per_ht = {str(args.ht): {"value": value, "ms_per_step": ms / args.steps,
                             "survivor_frac": surv_last / (BATCH * max(nloc, 1))}}
    for ht in [int(x) for x in args.per_ht.split(",") if x]:
        m2, _, _, s2 = timed(ht, max(3, args.steps // 2), 1)
        per_ht[str(ht)] = {"value": max(3, args.steps // 2) * BATCH * args.n / (m2 / 1e3),
                           "ms_per_step": m2 / max(3, args.steps // 2), "survivor_frac": s2 / (BATCH * max(nloc, 1))}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (K2 scan), from CUDA events around each launch
    pk, pk_kind = peaks()
    scan_ms, scan_n = scan
    avg = scan_ms / max(scan_n, 1)
    pairs = BATCH * nloc
    code_bytes = nloc * M  # algorithmic: each code read once per 256-query launch
    hbm_gbs = code_bytes / (avg / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "scan_ncu_summary.json")
    if os.path.exists(prof) and args.config == 1 and nloc == 100_000_000:
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": "hbm", "achieved": hbm_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": hbm_gbs / pk["hbm_gbs"], "traffic": traffic, "peak_kind": pk_kind,
                "kernel": f"K2 scan_kernel<{M},{16 if M == 8 else 8},{24 if M == 8 else 12},DUAL>", "kernel_ms_avg": avg,
                "kernel_launches": scan_n,
                "kernel_share_of_step": scan_ms / ms,
                "algorithmic_bytes_per_launch": code_bytes, "units_per_launch": f"{BATCH} queries x {nloc} codes"}
    # secondary roofline (the binding one for this integer/gather scan), per pair:
    #  m = 8 (tensor-core filter): TMEM read of the int32 D tile 4 B at 64 B/clk/SM, int8 MMA
    #    (6 x 8 clk per 4096 pairs), random LUT gathers 13.5/clk/SM (M per survivor);
    #  m = 16 (POPC filter): POPC 16/clk/SM (M/4 per pair) vs the same gathers.
    f_mhz = (clk or {}).get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    s = per_ht[str(args.ht)]["survivor_frac"]
    hbm_clk = float(M) / BATCH / (pk["hbm_gbs"] * 1e3 / f_mhz / 148)
    if M == 8:
        bound, clk_per_pair = "tmem-read/mma/lds-gather", max(4 / 64.0, 48 / 4096.0, s * M / 13.5, hbm_clk)
    else:
        bound, clk_per_pair = "popc/lds-gather", max(M / 4 / 16.0, s * M / 13.5, hbm_clk)
    peak_pairs = 148 * f_mhz * 1e6 / clk_per_pair
    # north_star's roofline: the slower of code bytes at HBM and the POPC / LUT-gather issue
    # rate of the Hamming test + ADC (an algorithmic bound: M/4 POPC per pair at 16/clk/SM)
    ns_clk = max(M / 4 / 16.0, s * M / 13.5, hbm_clk)
    ns_peak = 148 * f_mhz * 1e6 / ns_clk
    roofline_issue = {"bound": "popc/lds-gather issue (north_star)", "achieved": pairs / (avg / 1e3),
                      "peak": ns_peak, "unit": "pairs/s", "frac": pairs / (avg / 1e3) / ns_peak, "sm_mhz": f_mhz,
                      "clk_per_pair_bound": ns_clk, "survivor_frac": s}
    roofline_impl = {"bound": bound, "achieved": pairs / (avg / 1e3), "peak": peak_pairs,
                     "unit": "pairs/s", "frac": pairs / (avg / 1e3) / peak_pairs, "clk_per_pair_bound": clk_per_pair,
                     "note": "bound of the implemented kernel (m = 8: tensor-core filter, DESIGN.md 5)"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8/f32", "data": "synthetic (seeded Gaussian mixture, BASELINE cfg1)",
            "config": config(args, world), "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "roofline": roofline, "roofline_issue": roofline_issue, "roofline_impl": roofline_impl, "per_ht": per_ht,
            "setup_s": round(setup_s, 2)}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, index, hq.numpy())
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
