"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle on identical bytes.

Bar (BASELINE.json north_star): bit-exact Hamming distances, survivor sets,
query codes, database codes and top-k ids (ties included -- keys order by
(score, id) exactly); ADC scores are compared bit-exactly (tolerance 0), which
is stricter than the stated 1e-5 relative.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

TAUS8 = (0, 20, 24, 28, 32, 64)
TAUS16 = (0, 48, 56, 64, 128)


@pytest.fixture(scope="module")
def pb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1609_01882_b200 as pb
    return pb


def _index(pb, pq, codes=None, ids=None):
    ix = pb.FlatIndex(pb.ProductQuantizer(pq.m, pq.dbits, pq.dim, pq.codebooks, pq.perms))
    if codes is not None:
        ix.add_codes(codes, ids)
    return ix


def _same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


@pytest.mark.parametrize("which", ["8", "16"])
def test_lut_and_query_codes_bit_exact(pb, which, pq8, pq16, g8, g16):
    pq, g = (pq8, g8) if which == "8" else (pq16, g16)
    ix = _index(pb, pq)
    lutp, qc = pb.flat_index.debug_lut(ix, g["queries"])
    assert _same(qc, g["qcodes"])                                  # encode, pq.cpp:29-45
    assert _same(_bits(lutp[:4]), _bits(g["lutp"]))                # permuted_lut, pq.cpp:107-119


@pytest.mark.parametrize("which", ["8", "16"])
def test_gpu_encoder_matches_reference_encode(pb, which, pq8, pq16, g8, g16):
    pq, g = (pq8, g8) if which == "8" else (pq16, g16)
    centers = oracle.gen_centers(int(g["data_seed"]), int(g["ncent"]), pq.dim)
    base = oracle.gen_points(int(g["data_seed"]), 2, 0, int(g["n"]), centers)
    ix = _index(pb, pq)
    ix.add(base)
    assert ix.size() == base.shape[0]
    assert _same(ix.codes(), g["codes"])
    ix2 = _index(pb, pq)  # generated + encoded on the GPU, never materialised
    ix2.add_synthetic(int(g["data_seed"]), centers, 0, int(g["n"]))
    assert _same(ix2.codes(), g["codes"])
    assert _same(ix2.ids(), np.arange(int(g["n"])))


@pytest.mark.parametrize("strategy", ["adc", "binary", "disidx"])
@pytest.mark.parametrize("which", ["8", "16"])
def test_strategies_match_reference(pb, strategy, which, pq8, pq16, g8, g16):
    pq, g = (pq8, g8) if which == "8" else (pq16, g16)
    ix = _index(pb, pq, g["codes"])
    ids, sc, cnt = ix.search_batch(g["queries"], pb.SearchParams(pb.strategy_from_string(strategy), 100, 0))
    assert _same(ids, g[f"{strategy}_ids"])
    assert _same(_bits(sc), _bits(g[f"{strategy}_scores"]))
    assert _same(cnt, g[f"{strategy}_counts"])


@pytest.mark.parametrize("which", ["8", "16"])
def test_dual_matches_reference(pb, which, pq8, pq16, g8, g16):
    pq, g, taus = (pq8, g8, TAUS8) if which == "8" else (pq16, g16, TAUS16)
    ix = _index(pb, pq, g["codes"])
    nq = g["queries"].shape[0]
    for tau in taus:
        st = pb.SearchStats()
        ids, sc, cnt = ix.search_batch(g["queries"], pb.SearchParams(pb.Strategy.dual, 100, tau), st)
        assert _same(ids, g[f"dual{tau}_ids"]), tau
        assert _same(_bits(sc), _bits(g[f"dual{tau}_scores"])), tau
        assert _same(cnt, g[f"dual{tau}_counts"]), tau
        assert st.scanned == nq * g["codes"].shape[0]
        assert st.survivors == int(g[f"dual{tau}_surv"].sum()), tau


@pytest.mark.parametrize("which", ["8", "16"])
def test_ties_shortage_and_arbitrary_ids(pb, which, pq8, pq16, g8, g16):
    pq, g, taus = (pq8, g8, TAUS8) if which == "8" else (pq16, g16, TAUS16)
    tie_codes = np.repeat(g["codes"][:500], 4, axis=0)
    ix = _index(pb, pq, tie_codes, g["tie_ids_in"])
    for tau in (taus[1], pq.code_bits):
        ids, sc, cnt = ix.search_batch(g["queries"], pb.SearchParams(pb.Strategy.dual, 7, tau))
        assert _same(ids, g[f"tie{tau}_ids"])
        assert _same(cnt, g[f"tie{tau}_counts"])
    # ids beyond 32 bits and negative ids go through the rank table
    big = g["tie_ids_in"] * 1_000_000_007 - 5_000_000_000
    ixb = _index(pb, pq, tie_codes, big)
    ids_o, sc_o, cnt_o, _, _ = oracle.search(pq, tie_codes, g["queries"], 9, tau=taus[2], ids=big)
    ids, sc, cnt = ixb.search_batch(g["queries"], pb.SearchParams(pb.Strategy.dual, 9, taus[2]))
    assert _same(ids, ids_o) and _same(_bits(sc), _bits(sc_o)) and _same(cnt, cnt_o)


def test_edge_cases(pb, pq8, g8):
    q = g8["queries"][:5]
    ix = _index(pb, pq8, g8["codes"])
    ids, sc, cnt = ix.search_batch(q, pb.SearchParams(pb.Strategy.dual, 0, 24))   # k = 0 -> empty
    assert ids.shape == (5, 0) and cnt.tolist() == [0] * 5
    empty = _index(pb, pq8)                                                         # empty index -> empty
    ids, sc, cnt = empty.search_batch(q, pb.SearchParams(pb.Strategy.dual, 10, 24))
    assert cnt.tolist() == [0] * 5 and (ids == -1).all() and np.isinf(sc).all()
    with pytest.raises(pb.PolyError) as e:                                          # tau > code_bits
        ix.search_batch(q, pb.SearchParams(pb.Strategy.dual, 10, 65))
    assert e.value.code == pb.Errc.invalid_argument
    # k > n, and a single-query search() returns Neighbor objects
    small = _index(pb, pq8, g8["codes"][:37])
    ids, sc, cnt = small.search_batch(q, pb.SearchParams(pb.Strategy.adc, 50, 0))
    oi, os_, oc, _, _ = oracle.search(pq8, g8["codes"][:37], q, 50, strategy="adc")
    assert _same(ids, oi) and _same(cnt, oc) and (cnt == 37).all()
    res = ix.search(q[0], pb.SearchParams(pb.Strategy.dual, 5, 24))
    assert [r.id for r in res] == g8["dual24_ids"][0, :5].tolist()
    # a query equal to a stored code's reconstruction ranks that code first
    recon = np.concatenate([pq8.codebooks[sq, pq8.inv_perms[sq, g8["codes"][123, sq]]] for sq in range(8)])
    res = ix.search(recon, pb.SearchParams(pb.Strategy.dual, 3, 0))
    assert res[0].score == 0.0 and g8["codes"][res[0].id].tobytes() == g8["codes"][123].tobytes()


def test_calibrate_and_with_assignments(pb, pq8, g8):
    ix = _index(pb, pq8, g8["codes"])
    for rate in (0.5, 0.9, 0.95, 0.99, 1e-9):
        assert ix.calibrate_threshold(g8["queries"], rate) == oracle.calibrate_threshold(pq8, g8["codes"],
                                                                                         g8["queries"], rate)
    ident = np.tile(np.arange(256, dtype=np.uint16), (8, 1))
    ix2 = ix.with_assignments(ident)
    assert _same(ix2.codes(), oracle.relabel_codes(pq8, ident, g8["codes"]))
    pq_id = oracle.PQ(8, 8, 128, pq8.codebooks, ident)
    # adc is pi-invariant: same ids and scores under the new assignment
    a = ix.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.adc, 20, 0))
    b = ix2.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.adc, 20, 0))
    assert _same(a[0], b[0]) and _same(_bits(a[1]), _bits(b[1]))
    oi, _, _, _, _ = oracle.search(pq_id, ix2.codes(), g8["queries"], 20, tau=20)
    assert _same(ix2.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.dual, 20, 20))[0], oi)


@pytest.fixture(scope="module")
def big8(pb, pq8):
    """1M-code database generated + encoded on the GPU, checked against the CPU oracle."""
    seed = 160901882
    centers = oracle.gen_centers(seed, 1000, 128)
    ix = _index(pb, pq8)
    ix.add_synthetic(seed, centers, 0, 1_000_000)
    codes = ix.codes()
    sample = np.random.default_rng(0).choice(1_000_000, 2000, replace=False)
    rows = np.stack([oracle.gen_points(seed, 2, int(r), 1, centers)[0] for r in sample])
    assert _same(codes[sample], oracle.encode(pq8, rows))
    queries = oracle.gen_points(seed, 3, 0, 300, centers)
    return ix, codes, queries


@pytest.mark.parametrize("tau", [20, 24, 28, 32, 64])
def test_million_codes_match_oracle(pb, pq8, big8, tau):
    ix, codes, queries = big8
    oi, osc, oc, osv, _ = oracle.search(pq8, codes, queries, 100, tau=tau, threads=16)
    st = pb.SearchStats()
    ids, sc, cnt = ix.search_batch(queries, pb.SearchParams(pb.Strategy.dual, 100, tau), st)
    assert _same(ids, oi)
    assert _same(_bits(sc), _bits(osc))
    assert _same(cnt, oc)
    assert st.survivors == int(osv.sum())


def test_device_api_and_sharded_merge(pb, pq8, big8):
    """Shards searched separately and merged by K3 == the unsharded search
    (the multi-GPU exchange, run on one device)."""
    import torch
    ix, codes, queries = big8
    k, tau, G = 100, 24, 4
    p = pb.SearchParams(pb.Strategy.dual, k, tau)
    want = ix.search_batch(queries, p)
    dq = torch.from_numpy(queries).cuda()
    n = codes.shape[0]
    keys = torch.empty((G, len(queries), k), dtype=torch.int64, device="cuda")
    cnts = torch.empty((G, len(queries)), dtype=torch.int32, device="cuda")
    surv = torch.zeros((G, len(queries)), dtype=torch.int64, device="cuda")
    bounds = np.linspace(0, n, G + 1).astype(np.int64)
    shards = []
    for s in range(G):
        sh = _index(pb, pq8, codes[bounds[s]:bounds[s + 1]], np.arange(bounds[s], bounds[s + 1]))
        sh.search_keys_device(dq, p, keys[s], cnts[s], surv[s])
        shards.append(sh)
    oid = torch.empty((len(queries), k), dtype=torch.int64, device="cuda")
    osc = torch.empty((len(queries), k), dtype=torch.float32, device="cuda")
    ocnt = torch.empty(len(queries), dtype=torch.int32, device="cuda")
    shards[0].merge_keys_device(keys, cnts, G, len(queries), k, oid, osc, ocnt)
    torch.cuda.synchronize()
    # per-query survivor counts (the per-query-stats scan variant) == oracle
    _, _, _, osv, _ = oracle.search(pq8, codes, queries, k, tau=tau, threads=16)
    assert _same(surv.sum(0).cpu().numpy().astype(np.uint64), osv)
    assert _same(oid.cpu().numpy(), want[0])
    assert _same(_bits(osc.cpu().numpy()), _bits(want[1]))
    assert _same(ocnt.cpu().numpy().astype(np.uint32), want[2])
    # device-resident search == host search
    did = torch.empty((len(queries), k), dtype=torch.int64, device="cuda")
    dsc = torch.empty((len(queries), k), dtype=torch.float32, device="cuda")
    ix.search_batch_device(dq, p, did, dsc)
    torch.cuda.synchronize()
    assert _same(did.cpu().numpy(), want[0])


def test_launches_are_counted(pb, pq8, g8):
    ix = _index(pb, pq8, g8["codes"])
    before = pb.launch_count()
    ix.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.dual, 10, 24))
    assert pb.launch_count() - before >= 4  # K1, K2, K3, ids


def test_cpp_mirror_matches_reference(pb, pq8, g8, tmp_path):
    """A C++ caller of include/poly_b200/flat_index.hpp gets the reference's answers."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1609_01882_b200")
    exe = str(tmp_path / "mirror")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "mirror_smoke.cpp"), "-L", libdir, "-lpoly_b200",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    cb, pm, blob = (str(tmp_path / f) for f in ("cb.bin", "perms.bin", "blob.bin"))
    pq8.codebooks.tofile(cb)
    pq8.perms.tofile(pm)
    with open(blob, "wb") as f:
        f.write(g8["codes"].tobytes())
        f.write(g8["queries"].astype(np.float32).tobytes())
    out = subprocess.run([exe, cb, pm, blob], capture_output=True, text=True, check=True).stdout.split("\n")
    assert out[0] == f"stats {20000 * 24} {int(g8['dual24_surv'].sum())}"
    for i in range(24):
        assert [int(x) for x in out[1 + i].split()] == g8["dual24_ids"][i, :10].tolist()
    assert out[25] == "error 1"  # errc::invalid_argument for tau > code_bits
    assert out[26] == f"tau95 {oracle.calibrate_threshold(pq8, g8['codes'], g8['queries'], 0.95)[0]}"


@pytest.fixture(scope="module")
def big16(pb, pq16):
    """500k 128-bit codes (config-3 mixture) generated + encoded on the GPU."""
    seed = 160901882
    centers = oracle.gen_centers(seed, 4096, 256)
    ix = _index(pb, pq16)
    ix.add_synthetic(seed, centers, 0, 500_000)
    codes = ix.codes()
    sample = np.random.default_rng(1).choice(500_000, 500, replace=False)
    rows = np.stack([oracle.gen_points(seed, 2, int(r), 1, centers)[0] for r in sample])
    assert _same(codes[sample], oracle.encode(pq16, rows))
    return ix, codes, oracle.gen_points(seed, 3, 0, 160, centers)


@pytest.mark.parametrize("tau,strategy", [(48, "dual"), (56, "dual"), (64, "dual"), (0, "adc"), (0, "binary")])
def test_wide_codes_match_oracle(pb, pq16, big16, tau, strategy):
    ix, codes, queries = big16
    oi, osc, oc, osv, _ = oracle.search(pq16, codes, queries, 100, tau=tau, strategy=strategy, threads=16)
    st = pb.SearchStats()
    ids, sc, cnt = ix.search_batch(queries, pb.SearchParams(pb.strategy_from_string(strategy), 100, tau), st)
    assert _same(ids, oi)
    assert _same(_bits(sc), _bits(osc))
    assert _same(cnt, oc)
    if strategy == "dual":
        assert st.survivors == int(osv.sum())


def test_sharded_search_over_nccl_world1(pb, pq8, big8):
    """ShardedSearch through a real NCCL process group (world size 1 on one GPU):
    keys -> ncclAllGather -> K3 merge == the plain search."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_1609_01882_b200.distributed import FlatIndexEngine, ShardedSearch
    ix, codes, queries = big8
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        p = pb.SearchParams(pb.Strategy.dual, 100, 24)
        sharded = ShardedSearch(FlatIndexEngine(ix), device="cuda")
        sharded.world = 2  # exercise the all-gather + multi-part merge path with one rank's data twice
        dq = torch.from_numpy(queries).cuda()
        with pytest.raises(Exception):
            sharded.search_batch(dq, p)  # a world-1 group cannot gather 2 parts: fails loudly
        sharded.world = 1
        ids, sc, cnt = sharded.search_batch(dq, p)
        torch.cuda.synchronize()
        want = ix.search_batch(queries, p)
        assert _same(ids.cpu().numpy(), want[0])
        assert _same(_bits(sc.cpu().numpy()), _bits(want[1]))
        # the multi-part merge on duplicated parts keeps every id once per part: ties broken by id
        keys = torch.empty((len(queries), 100), dtype=torch.int64, device="cuda")
        kc = torch.empty(len(queries), dtype=torch.int32, device="cuda")
        ix.search_keys_device(dq, p, keys, kc)
        out = torch.empty((2 * len(queries), 100), dtype=torch.int64, device="cuda")
        dist.all_gather_into_tensor(out[:len(queries)], keys)
        torch.cuda.synchronize()
        assert torch.equal(out[:len(queries)], keys)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("parts,k,dist", [(1, 100, "spread"), (4, 1024, "narrow"), (6, 1000, "spread"),
                                          (64, 2048, "narrow"), (40, 500, "ties"), (3, 2048, "ties")])
def test_topk_select_paths(pb, pq8, parts, k, dist):
    """K3 through the merge entry point: direct sort (<= 2048 keys), bucket select from
    shared memory (<= 8192) or L2 (more), and the fallbacks when the k-th bucket is dense
    (many equal scores). Exact (score, id) order against numpy."""
    import torch
    rng = np.random.default_rng(parts * 7919 + k)
    nq = 5
    ix = _index(pb, pq8)
    if dist == "spread":
        sc = rng.uniform(0.0, 1e6, (parts, nq, k)).astype(np.float32)
    elif dist == "narrow":
        sc = rng.uniform(1000.0, 1001.0, (parts, nq, k)).astype(np.float32)
    else:
        sc = np.where(rng.random((parts, nq, k)) < 0.9, np.float32(7.5),
                      rng.uniform(7.0, 8.0, (parts, nq, k))).astype(np.float32)
    ranks = np.stack([rng.permutation(10_000_000)[:parts * k] for _ in range(nq)], 1)  # distinct per query
    ranks = ranks.reshape(parts, k, nq).transpose(0, 2, 1).astype(np.uint64)
    counts = rng.integers(k // 2, k + 1, (parts, nq)).astype(np.uint32)
    keys = (sc.view(np.uint32).astype(np.uint64) << np.uint64(32)) | ranks
    for p in range(parts):
        for q in range(nq):
            keys[p, q, counts[p, q]:] = np.uint64(0xFFFFFFFFFFFFFFFF)  # beyond the count: never read
    dk = torch.from_numpy(keys.reshape(-1).view(np.int64)).cuda()
    dc = torch.from_numpy(counts.reshape(-1).view(np.int32)).cuda()
    ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    scs = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    ix.merge_keys_device(dk, dc, parts, nq, k, ids, scs, cnt)
    torch.cuda.synchronize()
    for q in range(nq):
        allk = np.concatenate([keys[p, q, :counts[p, q]] for p in range(parts)])
        want = np.sort(allk)[:k]
        assert int(cnt[q]) == min(k, allk.size)
        assert np.array_equal(ids[q].cpu().numpy()[:want.size], (want & np.uint64(0xFFFFFFFF)).astype(np.int64))
        assert np.array_equal(_bits(scs[q].cpu().numpy()[:want.size]), (want >> np.uint64(32)).astype(np.uint32))


@pytest.mark.parametrize("n", [16_400, 20_000, 25_700, 33_000, 70_000])
def test_seed_sample_sizes_match_oracle(pb, pq8, g8, n):
    """DB sizes around the K2s seed sample (runs of 256 codes, at most n / 256 of them):
    the seeded bound must never drop a true top-k member (a code sampled twice would)."""
    codes = np.concatenate([g8["codes"]] * (n // g8["codes"].shape[0] + 1))[:n]
    ids = np.arange(n, dtype=np.int64) * 3 + 11
    ix = _index(pb, pq8, codes, ids)
    for tau in (20, 24, 32):
        want_ids, want_sc, want_cnt, want_surv, _ = oracle.search(pq8, codes, g8["queries"][:64], 100, tau=tau,
                                                                  ids=ids, threads=16)
        got_ids, got_sc, got_cnt = ix.search_batch(g8["queries"][:64], pb.SearchParams(pb.Strategy.dual, 100, tau))
        assert _same(got_ids, want_ids), (n, tau)
        assert _same(_bits(got_sc), _bits(want_sc)), (n, tau)
        assert _same(got_cnt, want_cnt), (n, tau)


def test_full_config1_size(pb, pq8):
    """BASELINE config 1 at its full size: N = 1e8 codes (generated + encoded on the GPU),
    one 256-query batch at tau = 24.  Exact against the oracle (the reference two-pass
    dual) for 8 queries over all 1e8 codes; for all 256 queries, size-independent checks
    of every returned neighbour: Hamming(code, qcode) <= tau, score == the fp32 ADC of its
    code (sq order), ascending (score, id) keys, counts = min(k, survivors)."""
    import os as _os
    seed = 160901882
    centers = oracle.gen_centers(seed, 1000, 128)
    ix = _index(pb, pq8)
    ix.add_synthetic(seed, centers, 0, 100_000_000)
    queries = oracle.gen_points(seed, 3, 0, 256, centers)
    tau, k = 24, 100
    ids, sc, cnt = ix.search_batch(queries, pb.SearchParams(pb.Strategy.dual, k, tau))
    codes = ix.codes()  # 800 MB on the host
    sub = np.array([0, 1, 37, 101, 128, 199, 254, 255])
    st = pb.SearchStats()
    ids_s, sc_s, cnt_s = ix.search_batch(queries[sub], pb.SearchParams(pb.Strategy.dual, k, tau), st)
    oi, osc, oc, osv, osh = oracle.search(pq8, codes, queries[sub], k, tau=tau, threads=_os.cpu_count() or 8)
    assert _same(ids_s, oi) and _same(ids[sub], oi)
    assert _same(_bits(sc_s), _bits(osc)) and _same(_bits(sc[sub]), _bits(osc))
    assert _same(cnt_s, oc) and _same(cnt[sub], oc)
    assert st.survivors == int(osv.sum())
    # survivor sets of the 8 queries over all 1e8 codes: per-query count and id hash
    import torch
    dq = torch.from_numpy(queries[sub]).cuda()
    did = torch.empty((len(sub), k), dtype=torch.int64, device="cuda")
    dsc = torch.empty((len(sub), k), dtype=torch.float32, device="cuda")
    sv = torch.empty(len(sub), dtype=torch.int64, device="cuda")
    sh = torch.empty(len(sub), dtype=torch.int64, device="cuda")
    ix.search_batch_device(dq, pb.SearchParams(pb.Strategy.dual, k, tau), did, dsc, None, sv,
                           stream=torch.cuda.current_stream().cuda_stream, d_survivor_hash=sh)
    torch.cuda.synchronize()
    assert _same(sv.cpu().numpy().view(np.uint64), osv)
    assert _same(sh.cpu().numpy().view(np.uint64), osh)
    # every returned neighbour of every query
    lutp, qc = pb.flat_index.debug_lut(ix, queries)
    assert (cnt == k).all()  # 1e8 codes: every query has >= k survivors
    rows = codes[ids]                                            # [256, k, 8]
    ham = np.unpackbits(rows ^ qc[:, None, :], axis=2).sum(2)
    assert (ham <= tau).all()
    acc = np.zeros(ids.shape, np.float32)
    for s in range(8):
        acc = (acc + np.take_along_axis(lutp[:, s, :], rows[:, :, s].astype(np.int64), axis=1)).astype(np.float32)
    assert _same(_bits(acc), _bits(sc))
    keys = (_bits(sc).astype(np.uint64) << np.uint64(32)) | ids.astype(np.uint64)
    assert (keys[:, 1:] > keys[:, :-1]).all()  # strictly ascending (score, id)


def test_full_config3_size(pb, pq16):
    """BASELINE config 3 at its full size: N = 2e8 128-bit codes (m = 16, POPC filter),
    tau = 56.  Exact against the oracle for 4 queries over all 2e8 codes; every returned
    neighbour of a 64-query batch satisfies the Hamming bound and carries the exact ADC."""
    import os as _os
    seed = 160901882
    centers = oracle.gen_centers(seed, 4096, 256)
    ix = _index(pb, pq16)
    ix.add_synthetic(seed, centers, 0, 200_000_000)
    queries = oracle.gen_points(seed, 3, 0, 64, centers)
    tau, k = 56, 100
    ids, sc, cnt = ix.search_batch(queries, pb.SearchParams(pb.Strategy.dual, k, tau))
    codes = ix.codes()  # 3.2 GB on the host
    sub = np.array([0, 17, 42, 63])
    oi, osc, oc, _, _ = oracle.search(pq16, codes, queries[sub], k, tau=tau, threads=_os.cpu_count() or 8)
    assert _same(ids[sub], oi)
    assert _same(_bits(sc[sub]), _bits(osc))
    assert _same(cnt[sub], oc)
    lutp, qc = pb.flat_index.debug_lut(ix, queries)
    rows = codes[ids]
    assert (np.unpackbits(rows ^ qc[:, None, :], axis=2).sum(2) <= tau).all()
    acc = np.zeros(ids.shape, np.float32)
    for s in range(16):
        acc = (acc + np.take_along_axis(lutp[:, s, :], rows[:, :, s].astype(np.int64), axis=1)).astype(np.float32)
    assert _same(_bits(acc), _bits(sc))


@pytest.mark.parametrize("seed", range(40))
def test_randomized_against_oracle(pb, pq8, pq16, g8, g16, seed):
    """Randomised sweep (sizes around tiles, seed runs, warm-up gates, batches and
    groups; k, tau, strategy, m, id schemes) of the flat search against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    wide = seed % 3 == 2
    pq, g = (pq16, g16) if wide else (pq8, g8)
    n = int(rng.choice([1, 7, 255, 256, 1535, 1536, 1537, 16385, 20000, 33000, 70000, 150000]))
    nq = int(rng.choice([1, 15, 16, 17, 100, 257, 300]))
    k = int(rng.choice([1, 10, 100, 257]))
    strategy = ["dual", "dual", "dual", "adc", "binary", "disidx"][seed % 6]
    tau = int(rng.integers(0, pq.code_bits + 1)) if strategy == "dual" else 0
    base = g["codes"]
    codes = base[rng.integers(0, base.shape[0], n)]
    id_mode = seed % 4
    if id_mode == 0:
        ids = None                                                   # positions
    elif id_mode == 1:
        ids = np.arange(n, dtype=np.int64) + 5_000_000_000          # arithmetic, above 2^32
    elif id_mode == 2:
        ids = rng.permutation(n).astype(np.int64) * 7 + 3           # arbitrary, not monotone
    else:
        ids = np.arange(n, dtype=np.int64) * 2                      # not consecutive
    qsrc = g["queries"]
    queries = qsrc[rng.integers(0, qsrc.shape[0], nq)] + rng.normal(0, 0.01, (nq, qsrc.shape[1])).astype(np.float32)
    queries = np.abs(queries).astype(np.float32)
    ix = _index(pb, pq, codes, ids)
    oi, osc, oc, osv, _ = oracle.search(pq, codes, queries, k, tau=tau, strategy=strategy,
                                        ids=np.arange(n, dtype=np.int64) if ids is None else ids, threads=16)
    st = pb.SearchStats()
    gi, gsc, gc = ix.search_batch(queries, pb.SearchParams(pb.strategy_from_string(strategy), k, tau), st)
    ctx = (n, nq, k, strategy, tau, wide, id_mode)
    assert _same(gi, oi), ctx
    assert _same(_bits(gsc), _bits(osc)), ctx
    assert _same(gc, oc), ctx
    if strategy == "dual" and tau < pq.code_bits:
        assert st.survivors == int(osv.sum()), ctx
