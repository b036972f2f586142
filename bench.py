#!/usr/bin/env python
"""Polysemous search on B200 -- the BASELINE.json headline metric, "DB codes scanned/sec
(filter+ADC+top-k)", on the BASELINE.json configurations.

    python bench.py [--gpus N --steps K --warmup W] [--config C] [--impl reference]

Configs (BASELINE.json "configs"; seeded synthetic data of the stated shapes and value
distributions -- DESIGN.md "Data"):
  0  flat, 64-bit codes, N = 1e6, nq = 1000, ht 24 (20/28/32/64 under per_ht)
  1  flat, 64-bit codes, N = 1e8 (800 MB), nq = 10,000 in batches of 256, ht 24 (28/32)
     -- the default: the configuration the metric is quoted on
  2  IVF 65,536 lists + 64-bit residual codes, N = 1e9 codes over the ranks, nq = 10,000
     (one step = all 10,000 queries), nprobe 16 (64 under per_nprobe), ht 26
  3  flat, 128-bit codes (m = 16), N = 2e8, ht 56 (48/64/128)
  4  k-NN graph: 1e7 unit vectors, IVF 16,384 + m = 16, nprobe 32, ht 52, k = 10

A step is one query batch through the whole path (flat: K1 LUT + query code, K2s seed,
K2 fused filter/ADC/candidate scan, K3 top-k, id map; IVF: coarse quantization, residual
LUTs, two K6 list-scan rounds, K3).  At N > 1 ranks the database is sharded (flat: id
ranges; IVF: ids within every list, the coarse quantization split by query) and the
per-rank top-k keys are all-gathered over NCCL and merged by K3.

`value` = codes scanned per second over the whole job, queries resident in HBM; time on
the device (CUDA events on the launching stream), max over ranks.  `e2e` = the same
metric through the library's host-buffer C-ABI call (poly_b200_search_batch /
poly_b200_ivf_search: queries copied from pinned host memory, results copied back, every
step).  `roofline` = the binding term of SURVEY.md sec. 8(d) for the dominant kernel
(K2 flat, K6 IVF): the slowest of code bytes at HBM bandwidth, POPC issue and LUT-gather
issue, at the SM clock sampled during the run; `roofline_step` adds the query-side FP32
(LUT builds) and TF32 (coarse quantization) terms for the whole step.  `cpu_baseline` =
the reference's CPU search (oracle/_ref: the reference's sources compiled in place) on a
bounded sample of the same workload, all host threads, plus a one-thread line.

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself under
torch.distributed.run with N ranks (one per GPU) and the NCCL INIT log on stderr.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
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
NQ = 10_000
CONFIGS = {
    0: dict(kind="flat", dim=128, ncent=1000, m=8, n=1_000_000, nq=1000, batch=256, ht=24, per_ht="20,28,32,64",
            pq="pq_d128_m8.npz", cpu_q=1000, cpu_q1=32),
    1: dict(kind="flat", dim=128, ncent=1000, m=8, n=100_000_000, nq=NQ, batch=256, ht=24, per_ht="28,32",
            pq="pq_d128_m8.npz", cpu_q=256, cpu_q1=4),
    2: dict(kind="ivf", dim=128, ncent=1000, m=8, n=1_000_000_000, nq=NQ, batch=NQ, ht=26, nlist=65536,
            nprobe=16, per_nprobe="64", pq="pq_ivf65536_d128_m8.npz", cpu_q=1000, cpu_q1=64),
    3: dict(kind="flat", dim=256, ncent=4096, m=16, n=200_000_000, nq=NQ, batch=256, ht=56, per_ht="48,64,128",
            pq="pq_d256_m16.npz", cpu_q=64, cpu_q1=2),
    4: dict(kind="knn", dim=256, ncent=4096, m=16, n=10_000_000, batch=2048, ht=52, nlist=16384, nprobe=32,
            knn_k=10, pq="pq_ivf16384_d256_m16.npz", cpu_q=10_000, cpu_q1=500),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=None, help="total database codes over all ranks (default: the config's N)")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--ht", type=int, default=None)
    ap.add_argument("--per-ht", default=None)
    ap.add_argument("--nprobe", type=int, default=None)
    ap.add_argument("--per-nprobe", default=None)
    ap.add_argument("--batch", type=int, default=None, help="queries per step (default: the config's batch)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-n", type=int, default=8_000_000, help="codes in each --impl reference step's sample")
    ap.add_argument("--spawn-check", action="store_true", help="launch/rendezvous self-test (CPU, gloo); tests only")
    ap.add_argument("--coarse", default="sample", choices=["sample", "kmeans"],
                    help="IVF coarse quantizer: training-stream rows (default) or GPU k-means (poly_b200_kmeans, "
                         "k-means++ + 10 Lloyd iterations on 16 x nlist training rows)")
    ap.add_argument("--ivf-shard", default="id", choices=["id", "list"],
                    help="multi-GPU IVF (config 2): shard ids within every list, or whole lists (assign_lists)")
    ap.add_argument("--knn-full", default=None, metavar="PATH",
                    help="config 4: also build this rank's whole k-NN graph into PATH (graph file sink, timed)")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config])
    args.c = c
    args.n = c["n"] if args.n is None else args.n
    args.k = (c.get("knn_k", 100)) if args.k is None else args.k
    args.ht = c["ht"] if args.ht is None else args.ht
    args.per_ht = c.get("per_ht", "") if args.per_ht is None else args.per_ht
    args.nprobe = c.get("nprobe", 0) if args.nprobe is None else args.nprobe
    args.per_nprobe = c.get("per_nprobe", "") if args.per_nprobe is None else args.per_nprobe
    args.batch = c["batch"] if args.batch is None else args.batch
    return args


# ------------------------------------------------------------------ launch
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args):
    """Re-run this script under torch.distributed.run, one rank per GPU."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # keep the communicator log visible ...
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr; stdout carries the JSON line
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def spawn_check(rank, world):
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.tensor([rank], dtype=torch.int64)
    out = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(out, t)
    if rank == 0:
        print(json.dumps({"spawn_check": True, "n_gpus": world, "ranks": [int(x.item()) for x in out]}), flush=True)
    dist.destroy_process_group()


# ------------------------------------------------------------------ measurement helpers
def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:  # B200_PROFILING.md fallback
        return {"hbm_gbs": 6650.0, "bf16_tflops": 2250.0, "sm_max_mhz": 1965.0}, "fallback"


def rates():
    """Per-SM-per-clock issue rates measured by tools/microbench.cu on the box
    (profiles/microbench.json): POPC, random 8 KB-table LDS gathers, packed FP32."""
    d = {"popc": 16.0, "lds_gather": 13.5, "fp32x2_ops": 256.0, "source": "defaults"}
    try:
        with open(os.path.join(ROOT, "profiles", "microbench.json")) as f:
            m = json.load(f)
        d.update({k: float(m[k]) for k in ("popc", "lds_gather", "fp32x2_ops") if k in m})
        d["source"] = "profiles/microbench.json"
    except (OSError, ValueError, KeyError):
        pass
    return d


def cpu_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "threads": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}


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
        if not sm:  # a timed region shorter than the 100 ms sampling period: one sample right after it
            try:
                f = subprocess.run(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                   capture_output=True, text=True, timeout=30).stdout.splitlines()[0].split(",")
                sm, smax = [float(f[1])], [float(f[2])]
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                reasons = {n for n, v in zip(names, f[5:9]) if v.strip().lower().startswith("active")}
            except (OSError, IndexError, ValueError, subprocess.SubprocessError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _clk(clk, pk):
    return (clk or {}).get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)


def scan_terms(m, reuse, survivor_frac, f_mhz, hbm_gbs, rt, filt=True, nsm=148):
    """SURVEY.md sec. 8(d) per-pair terms (clocks per pair per SM) of a scan over m-byte
    codes: code bytes at HBM bandwidth (each code read once per `reuse` queries), POPC
    (code_bits / 32 per pair; none when the filter keeps everything) and LUT gathers: m / 2
    per survivor -- the fewest any exact ADC can do here, since the half-sum early exit
    (code_ops.cuh adc_bounded) stops after m / 2 terms when the bound is exceeded (the
    full m per survivor of SURVEY.md sec. 8(d) is a looser bound: the plain-ADC kernel
    beats it)."""
    bytes_per_clk_sm = hbm_gbs * 1e9 / (nsm * f_mhz * 1e6)
    return {"hbm": m / reuse / bytes_per_clk_sm,
            "popc": (m * 8 / 32) / rt["popc"] if filt else 0.0,
            "lds": survivor_frac * (m / 2) / rt["lds_gather"]}


def roofline_from_terms(terms, achieved, f_mhz, nsm=148, unit="pairs/s"):
    bound = max(terms, key=terms.get)
    peak = nsm * f_mhz * 1e6 / terms[bound]
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "sm_mhz": f_mhz, "clk_per_pair": {k: round(v, 5) for k, v in terms.items()}}


# ------------------------------------------------------------------ reference arm
def run_reference(args, rank):
    """The reference's own CPU search (oracle/_ref: reference sources compiled in place;
    FlatIndex::search restated per SPEC from its primitives), all host threads.  Does not
    import the CUDA package: codes come from the reference's encode_batch on the CPU."""
    if rank != 0:
        return
    c = args.c
    if c["kind"] != "flat":
        print(json.dumps({"impl": "reference", "unavailable": f"config {args.config} needs a {args.n:.0e}-code IVF "
                          "database that only the GPU encoder builds in bench time; the reference CPU search is timed "
                          "on the real lists as cpu_baseline in the repo arm's line"}), flush=True)
        return
    import oracle
    threads = os.cpu_count()
    z = np.load(os.path.join(ROOT, "tests", "golden", c["pq"]))
    pq = oracle.PQ(c["m"], 8, c["dim"], z["codebooks"], z["perms"])
    kind = "reference" if oracle.ref_available() else "port"
    centers = oracle.gen_centers(SEED, c["ncent"], c["dim"])
    nsamp = min(args.ref_n, args.n)
    t = time.time()
    codes = np.empty((nsamp, c["m"]), np.uint8)
    step = 1 << 20
    for r0 in range(0, nsamp, step):
        x = oracle.gen_points(SEED, 2, r0, min(step, nsamp - r0), centers)
        codes[r0:r0 + len(x)] = oracle.ref_encode_batch(pq, x, threads) if kind == "reference" else oracle.encode(pq, x, threads)
    setup = time.time() - t
    nq = c["nq"]
    queries = oracle.gen_points(SEED, 3, 0, nq, centers)
    B = args.batch
    nb = max(1, nq // B)

    def search(q, thr):
        if kind == "reference":
            oracle.ref_search(pq, codes, q, args.k, tau=args.ht, threads=thr)
        else:
            oracle.search(pq, codes, q, args.k, tau=args.ht, threads=thr)

    for i in range(args.warmup):
        search(queries[(i % nb) * B:][:B], threads)
    t = time.perf_counter()
    for i in range(args.steps):
        search(queries[((args.warmup + i) % nb) * B:][:B], threads)
    dt = time.perf_counter() - t
    value = args.steps * B * nsamp / dt
    q1 = queries[:c["cpu_q1"]]
    t = time.perf_counter()
    search(q1, 1)
    dt1 = time.perf_counter() - t
    sample = (f"each step: {B} queries x the first {nsamp} codes of the cfg{args.config} database (of N={args.n}; "
              f"encoded by the reference's encode_batch), two-pass dual search, ht={args.ht}, k={args.k}; "
              f"{threads} threads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8/f32",
            "data": "synthetic (seeded Gaussian mixture; N(0,1) as Irwin-Hall(12) over splitmix64, DESIGN.md sec. 3)",
            "config": flat_config(args, 1, n_scanned=nsamp), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                             "cpu": cpu_info(),
                             "single_core": {"value": len(q1) * nsamp / dt1, "unit": UNIT, "cores": 1,
                                             "sample": f"{len(q1)} queries x {nsamp} codes, 1 thread"}},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": round(setup, 1)}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ flat (configs 0, 1, 3)
def flat_config(args, world, n_scanned=None):
    c = args.c
    d = {"workload": f"cfg{args.config} flat polysemous: N={args.n} {8 * c['m']}-bit codes (m={c['m']}, nbits=8, "
                     f"d={c['dim']} mixture of {c['ncent']}), nq={c['nq']} in batches of {args.batch}, k={args.k}, "
                     f"ht={args.ht}",
         "n_codes": args.n, "m": c["m"], "nbits": 8, "dim": c["dim"], "k": args.k, "ht": args.ht,
         "batch": args.batch, "nq": c["nq"], "strategy": "dual", "parallelism": f"db-shard{world}",
         "l2": (f"inputs larger than L2 ({args.n * c['m'] / 1e6:.0f} MB of codes vs 126 MB L2); no flush needed"
                if args.n * c["m"] > 126e6 else
                f"{args.n * c['m'] / 1e6:.0f} MB of codes: L2-resident by design (BASELINE cfg0 is the reference's "
                "CPU-runnable size); no flush")}
    if n_scanned is not None:
        d["n_codes_scanned_per_query"] = n_scanned
    return d


def cpu_baseline_flat(args, codes, queries):
    """Reference CPU search (oracle/_ref) on a bounded sample of the workload: cpu_q queries
    over all N codes on every host thread, and cpu_q1 queries on one thread."""
    import oracle
    c = args.c
    z = np.load(os.path.join(ROOT, "tests", "golden", c["pq"]))
    pq = oracle.PQ(c["m"], 8, c["dim"], z["codebooks"], z["perms"])
    threads = os.cpu_count()
    kind = "reference" if oracle.ref_available() else "port"
    fn = oracle.ref_search if kind == "reference" else oracle.search
    q = queries[:c["cpu_q"]]
    t = time.perf_counter()
    fn(pq, codes, q, args.k, tau=args.ht, threads=threads)
    dt = time.perf_counter() - t
    q1 = queries[:c["cpu_q1"]]
    t = time.perf_counter()
    fn(pq, codes, q1, args.k, tau=args.ht, threads=1)
    dt1 = time.perf_counter() - t
    n = codes.shape[0]
    return {"value": len(q) * n / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{len(q)} queries x all {n} codes, two-pass dual ht={args.ht}, k={args.k}, {dt:.1f} s",
            "cpu": cpu_info(),
            "single_core": {"value": len(q1) * n / dt1, "unit": UNIT, "cores": 1,
                            "sample": f"{len(q1)} queries x all {n} codes, 1 thread, {dt1:.1f} s"}}


def run_flat(args, rank, world, local):
    import torch
    import paper_1609_01882_b200 as pb
    from paper_1609_01882_b200 import synth
    from paper_1609_01882_b200.distributed import FlatIndexEngine, ShardedSearch, shard_range
    c = args.c
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    z = np.load(os.path.join(ROOT, "tests", "golden", c["pq"]))
    pq = pb.ProductQuantizer(c["m"], 8, c["dim"], z["codebooks"], z["perms"])
    centers = synth.gen_centers(SEED, c["ncent"], c["dim"])
    row0, row1 = shard_range(args.n, world, rank)
    nloc = row1 - row0
    t = time.time()
    index = pb.FlatIndex(pq, device=local)
    index.add_synthetic(SEED, centers, row0, nloc)   # GPU generator + encoder, ids = global rows
    setup_s = time.time() - t

    nq, B, k, M, dim = c["nq"], args.batch, args.k, c["m"], c["dim"]
    dq = torch.empty((nq, dim), dtype=torch.float32, device="cuda")
    pb.gen_points_device(centers, SEED, 3, 0, nq, dq, device=local)
    hq = dq.cpu().pin_memory()
    nb = max(1, nq // B)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    o_ids = torch.empty((B, k), dtype=torch.int64, device="cuda")
    o_sc = torch.empty((B, k), dtype=torch.float32, device="cuda")
    o_cnt = torch.empty(B, dtype=torch.int32, device="cuda")
    sharded = ShardedSearch(FlatIndexEngine(index), device="cuda") if world > 1 else None

    def step(i, ht, q=None):
        qb = dq[(i % nb) * B:][:B] if q is None else q
        p = pb.SearchParams(pb.Strategy.dual, k, ht)
        if world == 1:
            index.search_batch_device(qb, p, o_ids, o_sc, o_cnt, None, stream=sptr)
        else:  # local shard scan, NCCL all-gather of top-k keys, K3 merge
            sharded.search_batch(qb, p, out=(o_ids, o_sc, o_cnt))

    def survivor_frac(ht):
        st = pb.SearchStats()
        index.search_batch_device(dq[:B], pb.SearchParams(pb.Strategy.dual, k, ht), o_ids, o_sc, o_cnt, None,
                                  stream=sptr, stats=st)
        return st.survivors / (B * max(nloc, 1)) if ht < 8 * M else 1.0

    def timed(ht, steps, warmup, profile=False):
        for i in range(warmup):
            step(i, ht)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        if profile:
            index.profile_enable(True)
        prof = os.environ.get("BENCH_PROFILE") == "1" and profile  # ncu --profile-from-start off
        if prof:
            torch.cuda.profiler.start()
        l0 = pb.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            step(warmup + i, ht)
        e1.record(stream)
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
        launches = pb.launch_count() - l0
        ms = e0.elapsed_time(e1)
        scan = index.profile_read() if profile else None
        if profile:
            index.profile_enable(False)
        if dist:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms, launches, scan

    # ---- headline (device-resident)
    clocks = ClockSampler([local] if world == 1 else list(range(world))) if rank == 0 else None
    ms, launches, scan = timed(args.ht, args.steps, args.warmup, profile=True)
    clk = clocks.stop() if clocks else None
    value = args.steps * B * args.n / (ms / 1e3)
    s_head = survivor_frac(args.ht)

    # ---- e2e
    e2e = None
    if not args.no_e2e:
        h2d, d2h = B * dim * 4, B * k * 12 + B * 4
        if world == 1:
            # the drop-in host call (poly_b200_search_batch): pinned queries in, results out, synchronous
            out = (torch.empty((B, k), dtype=torch.int64).pin_memory().numpy(),
                   torch.empty((B, k), dtype=torch.float32).pin_memory().numpy(),
                   torch.empty(B, dtype=torch.int32).pin_memory().numpy().view(np.uint32))
            hqn = hq.numpy()
            p = pb.SearchParams(pb.Strategy.dual, k, args.ht)
            for i in range(args.warmup):
                index.search_batch(hqn[(i % nb) * B:][:B], p, out=out)
            t = time.perf_counter()
            for i in range(args.steps):
                index.search_batch(hqn[((args.warmup + i) % nb) * B:][:B], p, out=out)
            e2e_ms = (time.perf_counter() - t) * 1e3
            via = "poly_b200_search_batch (C ABI, host buffers; each call returns with the results in host memory)"
        else:
            h_ids = torch.empty((B, k), dtype=torch.int64).pin_memory()
            h_sc = torch.empty((B, k), dtype=torch.float32).pin_memory()
            h_cnt = torch.empty(B, dtype=torch.int32).pin_memory()
            qdev = torch.empty((B, dim), dtype=torch.float32, device="cuda")

            def e2e_step(i):
                qdev.copy_(hq[(i % nb) * B:][:B], non_blocking=True)
                step(i, args.ht, q=qdev)
                if rank == 0:
                    h_ids.copy_(o_ids, non_blocking=True)
                    h_sc.copy_(o_sc, non_blocking=True)
                    h_cnt.copy_(o_cnt, non_blocking=True)

            for i in range(args.warmup):
                e2e_step(i)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(args.steps):
                e2e_step(args.warmup + i)
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms = e0.elapsed_time(e1)
            t = torch.tensor([e2e_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
            d2h = d2h if rank == 0 else 0
            via = "ShardedSearch.search_batch with pinned host queries in / results out (CUDA events, max over ranks)"
        e2e = {"value": args.steps * B * args.n / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps, "via": via}

    # ---- per-ht sweep (device-resident); the K2 kernel time of each ht
    per_ht = {str(args.ht): {"value": value, "ms_per_step": ms / args.steps, "survivor_frac": s_head}}
    for ht in [int(x) for x in args.per_ht.split(",") if x]:
        st = max(3, args.steps // 2)
        m2, _, sc2 = timed(ht, st, 1, profile=True)
        per_ht[str(ht)] = {"value": st * B * args.n / (m2 / 1e3), "ms_per_step": m2 / st,
                           "survivor_frac": survivor_frac(ht), "k2_ms": sc2[0] / max(sc2[1], 1)}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    pk, pk_kind = peaks()
    rt = rates()
    f = _clk(clk, pk)
    scan_ms, scan_n = scan
    avg = scan_ms / max(scan_n, 1)
    pairs = B * nloc
    for ht, d in per_ht.items():  # the binding sec. 8(d) term per ht (K2 alone)
        kms = avg if ht == str(args.ht) else d.pop("k2_ms")
        filt = int(ht) < 8 * M
        r = roofline_from_terms(scan_terms(M, B, d["survivor_frac"], f, pk["hbm_gbs"], rt, filt),
                                pairs / (kms / 1e3), f)
        d["roofline_frac"] = round(r["frac"], 4)
        d["roofline_bound"] = r["bound"]
    roofline = roofline_from_terms(scan_terms(M, B, s_head, f, pk["hbm_gbs"], rt, args.ht < 8 * M),
                                   pairs / (avg / 1e3), f)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "scan_ncu_summary.json")
    if args.config == 1 and nloc == 100_000_000 and os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    q_per_cta = 16 if M == 8 else 8
    roofline.update({"traffic": traffic, "peak_kind": f"{pk_kind} HBM; issue rates {rt['source']}",
                     "kernel": f"K2 scan_kernel<{M},{q_per_cta},{28 if M == 8 else 14},DUAL>", "kernel_ms_avg": avg,
                     "kernel_launches": scan_n, "kernel_share_of_step": scan_ms / ms, "survivor_frac": s_head,
                     "units_per_launch": f"{B} queries x {nloc} codes = {pairs} pairs"})
    code_bytes = nloc * M
    roofline_hbm = {"bound": "hbm", "achieved": code_bytes / (avg / 1e3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
                    "frac": code_bytes / (avg / 1e3) / 1e9 / pk["hbm_gbs"], "traffic": traffic,
                    "algorithmic_bytes_per_launch": code_bytes,
                    "note": "the non-binding HBM term: each code is read once per 256-query launch"}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8/f32", "data": f"synthetic (seeded Gaussian mixture, BASELINE cfg{args.config}; N(0,1) as Irwin-Hall(12) over splitmix64, DESIGN.md sec. 3)",
            "config": flat_config(args, world), "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "roofline": roofline, "roofline_hbm": roofline_hbm, "per_ht": per_ht, "setup_s": round(setup_s, 2)}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_flat(args, index.codes(), hq.numpy())
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# ------------------------------------------------------------------ IVF (configs 2 and 4)
def build_ivf_by_list(args, pb, torch, local, rank, world, coarse, centers, norm):
    """By-list shard of rank: every rank assigns all rows (pass 1: list sizes -> the same
    assign_lists table everywhere), then keeps the rows of the cells it owns (pass 2),
    with their global ids."""
    from paper_1609_01882_b200.distributed import assign_lists
    c = args.c
    z = np.load(os.path.join(ROOT, "tests", "golden", c["pq"]))
    pq = pb.ProductQuantizer(c["m"], 8, c["dim"], z["codebooks"], z["perms"])
    ivf = pb.IVFIndex(pq, coarse, device=local)
    torch.backends.cuda.matmul.allow_tf32 = True
    dc = torch.from_numpy(coarse).cuda()
    cn = (dc * dc).sum(1)
    chunk = 1 << 21
    xbuf = torch.empty((chunk, c["dim"]), dtype=torch.float32, device="cuda")
    cells = torch.empty(chunk, dtype=torch.int32, device="cuda")

    def chunks():
        for r in range(0, args.n, chunk):
            nb = min(chunk, args.n - r)
            x = xbuf[:nb]
            pb.gen_points_device(centers, SEED, 2, r, nb, x, device=local, normalize=norm)
            for b in range(0, nb, 16384):
                xs = x[b:b + 16384]
                cells[b:b + xs.shape[0]] = torch.argmin(torch.addmm(cn, xs, dc.T, alpha=-2.0), dim=1).to(torch.int32)
            yield r, x, cells[:nb]

    hist = torch.zeros(c["nlist"], dtype=torch.int64, device="cuda")
    for _, _, cl in chunks():
        hist += torch.bincount(cl.to(torch.int64), minlength=c["nlist"])
    owner = torch.from_numpy(assign_lists(hist.cpu().numpy(), world).astype(np.int64)).cuda()
    for r, x, cl in chunks():
        keep = torch.nonzero(owner[cl.to(torch.int64)] == rank).squeeze(1)
        if keep.numel():
            ivf.add_device_ids(x[keep].contiguous(), cl[keep].contiguous(), (keep.cpu().numpy() + r).astype(np.int64))
    ivf.list_offsets()
    torch.cuda.synchronize()
    return ivf, pq


def build_ivf(args, pb, torch, local, row0, row1, coarse, centers, norm):
    """GPU build of this rank's rows: generator, nearest-cell assignment (TF32 GEMM argmin
    through torch -- setup, not the measured path), exact residual encoding (C ABI)."""
    c = args.c
    z = np.load(os.path.join(ROOT, "tests", "golden", c["pq"]))
    pq = pb.ProductQuantizer(c["m"], 8, c["dim"], z["codebooks"], z["perms"])
    ivf = pb.IVFIndex(pq, coarse, device=local)
    torch.backends.cuda.matmul.allow_tf32 = True
    dc = torch.from_numpy(coarse).cuda()
    cn = (dc * dc).sum(1)
    chunk = 1 << 21
    xbuf = torch.empty((chunk, c["dim"]), dtype=torch.float32, device="cuda")
    cells = torch.empty(chunk, dtype=torch.int32, device="cuda")
    for r in range(row0, row1, chunk):
        nb = min(chunk, row1 - r)
        x = xbuf[:nb]
        pb.gen_points_device(centers, SEED, 2, r, nb, x, device=local, normalize=norm)
        for b in range(0, nb, 16384):
            xs = x[b:b + 16384]
            cells[b:b + xs.shape[0]] = torch.argmin(torch.addmm(cn, xs, dc.T, alpha=-2.0), dim=1).to(torch.int32)
        ivf.add_device(x, cells[:nb], r)
    ivf.list_offsets()  # CSR rebuild now (setup), not inside the first timed search
    torch.cuda.synchronize()
    return ivf, pq


def cpu_baseline_ivf(args, ivf, queries, nprobe, k, coarse, pq_host):
    """Reference CPU search_coarse (oracle/_ref ref_ivf_search: coarse sq_l2 over every
    cell, residual encode + LUT per probe, two-pass dual scan, corrected heap) on the
    real lists: only the probed cells' lists are copied to the host (the search visits
    no others), on every host thread and on one."""
    import oracle
    threads = os.cpu_count()
    kind = "reference" if oracle.ref_available() else "port"
    nlist = args.c["nlist"]
    queries = np.ascontiguousarray(queries, np.float32)
    probes = ivf.probes(queries, nprobe)                # exact enumerate_cells (the CPU computes the same)
    cells = np.unique(probes)
    off_c, codes, ids = ivf.cells(cells)
    sizes = np.zeros(nlist, np.uint64)
    sizes[cells] = np.diff(off_c)
    off = np.zeros(nlist + 1, np.uint64)
    off[1:] = np.cumsum(sizes)
    lists = oracle.IVFLists(off, codes, ids)            # cells ascending == np.unique order
    opq = oracle.PQ(pq_host.m, 8, pq_host.dim, pq_host.codebooks, pq_host.perms)
    scanned = int(sizes[probes].sum())
    fn = oracle.ref_ivf_search if kind == "reference" else oracle.ivf_search
    t = time.perf_counter()
    fn(opq, coarse, lists, queries, k, nprobe, tau=args.ht, threads=threads)
    dt = time.perf_counter() - t
    q1 = queries[:args.c["cpu_q1"]]
    scanned1 = int(sizes[probes[:len(q1)]].sum())
    t = time.perf_counter()
    fn(opq, coarse, lists, q1, k, nprobe, tau=args.ht, threads=1)
    dt1 = time.perf_counter() - t
    return {"value": scanned / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{len(queries)} queries, nprobe {nprobe}, k {k}, ht {args.ht}: {scanned} codes scanned, "
                      f"coarse quantization + residual LUTs + dual scan, {dt:.1f} s",
            "cpu": cpu_info(),
            "single_core": {"value": scanned1 / dt1, "unit": UNIT, "cores": 1,
                            "sample": f"{len(q1)} queries, 1 thread, {dt1:.1f} s"}}


def ivf_rooflines(args, pk, rt, f, m, scanned, surv, nq_step, np_step, ms_step, k6_ms, world):
    """K6 (dominant kernel) sec. 8(d) terms, and the whole step with the query-side terms
    (residual LUT builds at the measured packed-FP32 rate, coarse dots at half the
    measured bf16 tensor rate = TF32)."""
    s = surv / max(scanned, 1)
    terms = scan_terms(m, 1, s, f, pk["hbm_gbs"], rt)
    per_pair_s = {kk: v / (148 * f * 1e6) for kk, v in terms.items()}
    k6 = roofline_from_terms(terms, scanned / (k6_ms / 1e3), f)
    lut_ops = nq_step * np_step * m * 256 * 16 * 3               # sub, mul, add per (centroid, dim)
    coarse_flop = nq_step / world * args.c["nlist"] * args.c["dim"] * 2
    step_terms_s = {kk: v * scanned for kk, v in per_pair_s.items()}
    step_terms_s["fp32_lut"] = lut_ops / (rt["fp32x2_ops"] * 148 * f * 1e6)
    step_terms_s["tf32_coarse"] = coarse_flop / (pk.get("bf16_tflops", 1637.0) / 2 * 1e12)
    bound = max(step_terms_s, key=step_terms_s.get)
    t_min = step_terms_s[bound]
    step = {"bound": bound, "achieved": scanned / (ms_step / 1e3), "peak": scanned / t_min, "unit": "codes/s",
            "frac": t_min / (ms_step / 1e3), "terms_ms": {kk: round(v * 1e3, 4) for kk, v in step_terms_s.items()},
            "scope": "whole step (every kernel), per rank"}
    hbm = {"bound": "hbm", "achieved": scanned * m / (k6_ms / 1e3) / 1e9, "peak": pk["hbm_gbs"], "unit": "GB/s",
           "frac": scanned * m / (k6_ms / 1e3) / 1e9 / pk["hbm_gbs"], "algorithmic_bytes_per_step": scanned * m}
    return k6, step, hbm


def make_coarse(args, pb, synth, centers, norm):
    """The coarse quantizer: the first nlist training-stream rows (the fixtures' recipe), or
    GPU k-means (train_coarse) on 16 x nlist training rows, 10 Lloyd iterations."""
    c = args.c
    if args.coarse == "sample":
        return synth.gen_points(SEED, 1, 0, c["nlist"], centers, normalize=norm)
    t = time.time()
    train = synth.gen_points(SEED, 1, 0, 16 * c["nlist"], centers, normalize=norm)
    cent, _, _, mse = pb.kmeans(train, c["nlist"], iters=10, seed=1234567)
    args.coarse_info = {"kind": "kmeans", "train_rows": len(train), "iters": 10, "mse": mse,
                        "train_s": round(time.time() - t, 1)}
    return cent


def run_ivf(args, rank, world, local):
    """search_coarse throughput (config 2): codes scanned/s over the probed lists."""
    import torch
    import paper_1609_01882_b200 as pb
    from paper_1609_01882_b200 import synth
    from paper_1609_01882_b200.distributed import IVFIndexEngine, ShardedSearch, shard_range
    c = args.c
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    centers = synth.gen_centers(SEED, c["ncent"], c["dim"])
    coarse = make_coarse(args, pb, synth, centers, False)
    row0, row1 = shard_range(args.n, world, rank)
    t = time.time()
    if args.ivf_shard == "list":
        ivf, pq = build_ivf_by_list(args, pb, torch, local, rank, world, coarse, centers, False)
    else:
        ivf, pq = build_ivf(args, pb, torch, local, row0, row1, coarse, centers, False)
    setup_s = time.time() - t
    nq, B, k, M = c["nq"], args.batch, args.k, c["m"]
    ivf.set_batch(B)  # one internal batch per step: the cell-major scan groups the step's queries per list
    dq = torch.empty((nq, c["dim"]), dtype=torch.float32, device="cuda")
    pb.gen_points_device(centers, SEED, 3, 0, nq, dq, device=local)
    stream = torch.cuda.current_stream()
    o_ids = torch.empty((B, k), dtype=torch.int64, device="cuda")
    o_sc = torch.empty((B, k), dtype=torch.float32, device="cuda")
    o_cnt = torch.empty(B, dtype=torch.int32, device="cuda")
    nb = max(1, nq // B)
    # keys exchanged all-to-all by query slice: each rank merges 1/world of the queries
    sharded = ShardedSearch(IVFIndexEngine(ivf, split_coarse=True, by_list=args.ivf_shard == "list"),
                            exchange="alltoall") if dist else None

    def step(i, p, st=None):
        q = dq[(i % nb) * B:][:B]
        if dist is None:
            ivf.search_device(q, p, o_ids, o_sc, o_cnt, stream.cuda_stream, st)
        else:
            sharded.engine.stats = st
            sharded.search_batch(q, p, (o_ids, o_sc, o_cnt))

    results = {}
    clk = None
    for nprobe in [args.nprobe] + [int(x) for x in args.per_nprobe.split(",") if x]:
        p = pb.CoarseParams(pb.Strategy.dual, k, args.ht, nprobe, 0)
        steps = args.steps if nprobe == args.nprobe else max(3, args.steps // 2)
        scanned = surv = 0
        for i in range(args.warmup, args.warmup + steps):  # per-step work counts (untimed)
            st = pb.SearchStats()
            step(i, p, st)
            scanned += st.scanned
            surv += st.survivors
        if dist is not None:  # codes scanned by all ranks
            tt = torch.tensor([scanned, surv], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt)
            scanned_all = int(tt[0].item())
        else:
            scanned_all = scanned
        for i in range(args.warmup):
            step(i, p)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        head = nprobe == args.nprobe
        clocks = ClockSampler([local] if world == 1 else list(range(world))) if rank == 0 and head else None
        ivf.profile_enable(True)
        prof = os.environ.get("BENCH_PROFILE") == "1" and head
        if prof:
            torch.cuda.profiler.start()
        l0 = pb.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.warmup, args.warmup + steps):
            step(i, p)
        e1.record(stream)
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
        if clocks:
            clk = clocks.stop()
        ms = e0.elapsed_time(e1)
        k6_ms, _ = ivf.profile_read()
        ivf.profile_enable(False)
        if dist is not None:  # max over ranks
            tt = torch.tensor([ms], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt.item())
        results[nprobe] = {"value": scanned_all / (ms / 1e3), "ms_per_step": ms / steps,
                           "scanned_per_query": scanned / (steps * B), "survivor_frac": surv / max(scanned, 1),
                           "gpu_launches": pb.launch_count() - l0, "steps": steps,
                           "_local": (scanned / steps, surv / steps, k6_ms / steps, ms / steps)}

    # ---- e2e through the host-buffer call (N = 1): poly_b200_ivf_search
    e2e = None
    if not args.no_e2e and world == 1:
        hq = dq.cpu().pin_memory().numpy()
        out = (torch.empty((B, k), dtype=torch.int64).pin_memory().numpy(),
               torch.empty((B, k), dtype=torch.float32).pin_memory().numpy(),
               torch.empty(B, dtype=torch.int32).pin_memory().numpy().view(np.uint32))
        p = pb.CoarseParams(pb.Strategy.dual, k, args.ht, args.nprobe, 0)
        for i in range(args.warmup):
            ivf.search(hq[(i % nb) * B:][:B], p, out=out)
        t = time.perf_counter()
        for i in range(args.steps):
            ivf.search(hq[((args.warmup + i) % nb) * B:][:B], p, out=out)
        e2e_ms = (time.perf_counter() - t) * 1e3
        h = results[args.nprobe]
        e2e = {"value": h["value"] * h["ms_per_step"] * args.steps / e2e_ms, "unit": UNIT,
               "h2d_bytes_per_step": B * c["dim"] * 4, "d2h_bytes_per_step": B * k * 12 + B * 4,
               "ms_per_step": e2e_ms / args.steps,
               "via": "poly_b200_ivf_search (C ABI, host buffers; synchronous per call)"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    pk, _ = peaks()
    rt = rates()
    f = _clk(clk, pk)
    # by-list sharding at 8 ranks: per-rank share of the codes a step's
    # probes scan, cells placed by assign_lists on this index's list sizes (rank 0's shard)
    from paper_1609_01882_b200.distributed import assign_lists, by_list_balance
    sizes = np.diff(ivf.list_offsets().astype(np.int64))
    owner8 = assign_lists(sizes, 8)
    cells = ivf.probes(dq[:B].cpu().numpy(), args.nprobe).astype(np.int64)
    imb, per8 = by_list_balance(sizes, cells, owner8, 8)
    by_list = {"ranks": 8, "scan_imbalance_max_over_mean": round(imb, 4),
               "list_codes_imbalance": round(float(np.bincount(owner8, weights=sizes, minlength=8).max() /
                                                   max(sizes.sum() / 8, 1)), 4),
               "note": "codes the step's probes scan per rank under assign_lists (LPT by list size), max / mean"}
    for nprobe, r in results.items():
        sc_l, sv_l, k6_l, ms_l = r.pop("_local")
        k6, stp, hbm = ivf_rooflines(args, pk, rt, f, M, sc_l, sv_l, B, nprobe, ms_l, k6_l, world)
        r["roofline"], r["roofline_step"], r["roofline_hbm"] = k6, stp, hbm
        r["k6_share_of_step"] = k6_l / ms_l
    head = results[args.nprobe]
    line = {"metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": head["steps"],
            "warmup": args.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8/f32", "data": "synthetic (seeded Gaussian mixture, BASELINE cfg2; N(0,1) as Irwin-Hall(12) over splitmix64, DESIGN.md sec. 3)",
            "config": {"workload": f"cfg2 IVF+polysemous: nlist={c['nlist']}, N={args.n} codes over {world} GPU(s), "
                                   f"PQ m={M} on residuals, nq={nq} in batches of {B}, nprobe={args.nprobe}, k={k}, "
                                   f"ht={args.ht}",
                       "nlist": c["nlist"], "n_codes": args.n, "m": M, "nprobe": args.nprobe, "k": k, "ht": args.ht,
                       "batch": B, "parallelism": f"db-shard{world} ({'whole lists per rank (assign_lists)' if args.ivf_shard == 'list' else 'ids within every list'}) + query-split coarse "
                                                  "quantization + NCCL probe / key all-gathers",
                       "coarse": getattr(args, "coarse_info", "training-stream rows [0, nlist) (sampled coarse quantizer; DESIGN.md)"),
                       "build_assignment": "TF32 GEMM argmin (setup only)",
                       "l2": "probed lists stream from HBM (GBs of codes per GPU); no flush needed"},
            "e2e": e2e, "gpu_launches": head["gpu_launches"], "clocks": clk,
            "roofline": dict(head["roofline"], kernel="K6 ivf_list_scan_kernel (both rounds)",
                             kernel_share_of_step=head["k6_share_of_step"]),
            "roofline_step": head["roofline_step"], "roofline_hbm": head["roofline_hbm"],
            "by_list_sharding_8": by_list,
            "per_nprobe": {str(kk): {x: v for x, v in r.items() if x not in ("roofline_step", "roofline_hbm")}
                           for kk, r in results.items()},
            "setup_s": round(setup_s, 1)}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_ivf(args, ivf, dq[:c["cpu_q"]].cpu().numpy(), args.nprobe, k, coarse, pq)
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def knn_full(args, pb, torch, ivf, centers, p, row0, row1, local, stream):
    """The whole graph of rows [row0, row1) through the output sink (graph file + ivecs):
    rows generated on the GPU in 1M-row chunks, searched, written while the next step runs.
    Wall clock around the whole run (generation, search, copies, file writes)."""
    c = args.c
    chunk = 1 << 20
    dx = torch.empty((chunk, c["dim"]), dtype=torch.float32, device="cuda")
    path = args.knn_full
    t = time.perf_counter()
    with pb.KnnGraphWriter(path, p.k, path + ".ivecs") as w:
        for r in range(row0, row1, chunk):
            nb = min(chunk, row1 - r)
            pb.gen_points_device(centers, SEED, 2, r, nb, dx[:nb], device=local, normalize=True)
            ivf.knn_graph_write_device(w, dx[:nb], r, p, stream.cuda_stream)
    wall = time.perf_counter() - t
    rows = row1 - row0
    return {"rows": rows, "records": w.records, "wall_s": round(wall, 2), "rows_per_s": rows / wall,
            "file_bytes": os.path.getsize(path), "ivecs_bytes": os.path.getsize(path + ".ivecs"),
            "note": "knn_graph_write_device per 1M-row chunk; wall clock includes generation, copies, writes"}


def run_knn(args, rank, world, local):
    """Config 4: the k-NN graph.  A step = B stored vectors searched against the whole
    index with k + 1 neighbours and the self-match removed (knn_graph_device)."""
    import torch
    import paper_1609_01882_b200 as pb
    from paper_1609_01882_b200 import synth
    from paper_1609_01882_b200.distributed import shard_range
    c = args.c
    torch.cuda.set_device(local)
    centers = synth.gen_centers(SEED, c["ncent"], c["dim"])
    coarse = make_coarse(args, pb, synth, centers, True)
    t = time.time()
    ivf, pq = build_ivf(args, pb, torch, local, 0, args.n, coarse, centers, True)
    setup_s = time.time() - t
    row0, row1 = shard_range(args.n, world, rank)   # this rank's query rows (cfg4 shards the query set)
    k, B, M = args.k, args.batch, c["m"]
    ivf.set_batch(B)
    p = pb.CoarseParams(pb.Strategy.dual, k, args.ht, args.nprobe, 0)
    p1 = pb.CoarseParams(pb.Strategy.dual, k + 1, args.ht, args.nprobe, 0)
    stream = torch.cuda.current_stream()
    steps = args.steps
    nrows = (args.warmup + steps) * B
    dx = torch.empty((nrows, c["dim"]), dtype=torch.float32, device="cuda")
    pb.gen_points_device(centers, SEED, 2, row0, nrows, dx, device=local, normalize=True)
    o_ids = torch.empty((B, k), dtype=torch.int64, device="cuda")
    o_sc = torch.empty((B, k), dtype=torch.float32, device="cuda")
    o_cnt = torch.empty(B, dtype=torch.int32, device="cuda")
    ob = (torch.empty((B, k + 1), dtype=torch.int64, device="cuda"),
          torch.empty((B, k + 1), dtype=torch.float32, device="cuda"))
    scanned = surv = 0
    for i in range(args.warmup, args.warmup + steps):  # per-step work counts (untimed)
        st = pb.SearchStats()
        ivf.search_device(dx[i * B:(i + 1) * B], p1, ob[0], ob[1], None, stream.cuda_stream, st)
        scanned += st.scanned
        surv += st.survivors
    for i in range(args.warmup):
        ivf.knn_graph_device(dx[i * B:(i + 1) * B], row0 + i * B, p, o_ids, o_sc, o_cnt, stream.cuda_stream)
    torch.cuda.synchronize()
    clocks = ClockSampler([local]) if rank == 0 else None
    ivf.profile_enable(True)
    l0 = pb.launch_count()
    prof = os.environ.get("BENCH_PROFILE") == "1"  # ncu --profile-from-start off: the timed steps only
    if prof:
        torch.cuda.profiler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.warmup, args.warmup + steps):
        ivf.knn_graph_device(dx[i * B:(i + 1) * B], row0 + i * B, p, o_ids, o_sc, o_cnt, stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    if prof:
        torch.cuda.profiler.stop()
    clk = clocks.stop() if clocks else None
    launches = pb.launch_count() - l0
    ms = e0.elapsed_time(e1)
    k6_ms, _ = ivf.profile_read()
    ivf.profile_enable(False)
    # ---- e2e (N = 1): every step's rows come in from pinned host memory and its neighbours,
    # scores and counts go back out, around the same public call
    e2e = None
    if not args.no_e2e and world == 1:
        h_rows = torch.empty((nrows, c["dim"]), dtype=torch.float32).pin_memory()
        h_rows.copy_(dx)
        d_in = torch.empty((B, c["dim"]), dtype=torch.float32, device="cuda")
        h_ids = torch.empty((B, k), dtype=torch.int64).pin_memory()
        h_sc = torch.empty((B, k), dtype=torch.float32).pin_memory()
        h_cnt = torch.empty(B, dtype=torch.int32).pin_memory()

        def e2e_step(i):
            d_in.copy_(h_rows[i * B:(i + 1) * B], non_blocking=True)
            ivf.knn_graph_device(d_in, row0 + i * B, p, o_ids, o_sc, o_cnt, stream.cuda_stream)
            h_ids.copy_(o_ids, non_blocking=True)
            h_sc.copy_(o_sc, non_blocking=True)
            h_cnt.copy_(o_cnt, non_blocking=True)
            stream.synchronize()

        for i in range(args.warmup):
            e2e_step(i)
        t = time.perf_counter()
        for i in range(args.warmup, args.warmup + steps):
            e2e_step(i)
        e2e_ms = (time.perf_counter() - t) * 1e3
        e2e = {"value": scanned / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": B * c["dim"] * 4,
               "d2h_bytes_per_step": B * k * 12 + B * 4, "ms_per_step": e2e_ms / steps,
               "via": "poly_b200_ivf_knn_graph_device; the step's rows copied in from pinned host memory and its "
                      "ids / scores / counts copied out, synchronised every step"}
    if rank != 0:
        return
    pk, _ = peaks()
    rt = rates()
    f = _clk(clk, pk)
    k6, stp, hbm = ivf_rooflines(args, pk, rt, f, M, scanned / steps, surv / steps, B, args.nprobe, ms / steps,
                                 k6_ms / steps, 1)
    rows = row1 - row0
    line = {"metric": METRIC, "value": scanned / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8/f32", "data": "synthetic (unit-normalised mixture, BASELINE cfg4; N(0,1) as Irwin-Hall(12) over splitmix64, DESIGN.md sec. 3)",
            "config": {"workload": f"cfg4 k-NN graph: N={args.n} d={c['dim']} unit-normalised, IVF {c['nlist']} + PQ "
                                   f"m={M}, every vector queries the rest, nprobe={args.nprobe}, ht={args.ht}, k={k}",
                       "n_codes": args.n, "nlist": c["nlist"], "m": M, "nprobe": args.nprobe, "k": k,
                       "ht": args.ht, "queries_per_step": B,
                       "l2": "160 MB of list codes stream through L2 per step; no flush"},
            "scanned_per_query": scanned / (steps * B), "survivor_frac": surv / max(scanned, 1),
            "graph_time_est_s": rows / B * ms / steps / 1e3, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "roofline": dict(k6, kernel="K6 ivf_list_scan_kernel (both rounds)", kernel_share_of_step=k6_ms / ms),
            "roofline_step": stp, "roofline_hbm": hbm, "setup_s": round(setup_s, 1)}
    if args.knn_full:
        line["full_graph"] = knn_full(args, pb, torch, ivf, centers, p, row0, row1, local, stream)
    if world == 1 and not args.no_cpu_baseline:
        rng = np.random.default_rng(SEED)
        rows_s = np.sort(rng.choice(args.n, c["cpu_q"], replace=False))   # the seeded 10k-query subsample
        xq = np.concatenate([synth.gen_points(SEED, 2, int(r), 1, centers, normalize=True) for r in rows_s])
        line["cpu_baseline"] = cpu_baseline_ivf(args, ivf, xq, args.nprobe, k + 1, coarse, pq)
        line["cpu_baseline"]["sample"] += " (seeded 10k-row subsample of the graph's queries, k + 1 = 11)"
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.spawn_check:
        spawn_check(rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank)
        return
    kind = args.c["kind"]
    if kind == "flat":
        run_flat(args, rank, world, local)
    elif kind == "ivf":
        run_ivf(args, rank, world, local)
    else:
        run_knn(args, rank, world, local)


if __name__ == "__main__":
    main()
