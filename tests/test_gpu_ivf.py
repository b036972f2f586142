"""GPU parity of the IVF path through the C ABI: build,
enumerate_cells, search_coarse (nprobe, cap, tau, strategies) against golden
vectors composed from the reference's primitives and against the oracle.
Bit-exact: lists, probe order, ids, scores, counts, survivors."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_ivf.npz")


@pytest.fixture(scope="module")
def pb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1609_01882_b200 as pb
    return pb


@pytest.fixture(scope="module")
def gi():
    z = dict(np.load(GOLDEN))
    z["pq"] = oracle.PQ(8, 8, 128, z["codebooks"], z["perms"])
    z["lists"] = oracle.IVFLists(z["off"], z["list_codes"], z["list_ids"])
    return z


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def _ivf(pb, gi):
    pq = pb.ProductQuantizer(8, 8, 128, gi["codebooks"], gi["perms"])
    return pb.IVFIndex(pq, gi["coarse"])


@pytest.fixture(scope="module")
def built(pb, gi):
    centers = oracle.gen_centers(int(gi["data_seed"]), 1000, 128)
    base = oracle.gen_points(int(gi["data_seed"]), 2, 0, int(gi["n"]), centers)
    ix = _ivf(pb, gi)
    ix.add(base, ids=np.arange(int(gi["n"])) * 7 + 3)  # GPU assignment + residual encode
    return ix, base


def test_build_matches_reference(pb, gi, built):
    ix, base = built
    assert np.array_equal(ix.assign(base), gi["assign_exact"])
    off, codes, ids = ix.lists()
    assert np.array_equal(off, gi["off"])
    for c in range(len(off) - 1):  # order inside a list is not part of the contract
        a, b = int(off[c]), int(off[c + 1])
        og = np.argsort(gi["list_ids"][a:b])
        ob = np.argsort(ids[a:b])
        assert np.array_equal(ids[a:b][ob], gi["list_ids"][a:b][og])
        assert np.array_equal(codes[a:b][ob], gi["list_codes"][a:b][og])


def test_probe_order_matches_oracle(pb, gi, built):
    ix, _ = built
    for nprobe in (1, 7, 64):
        want = oracle.ivf_search(gi["pq"], gi["coarse"], gi["lists"], gi["queries"], 5, nprobe)[5]
        assert np.array_equal(ix.probes(gi["queries"], nprobe), want)


@pytest.mark.parametrize("nprobe", [1, 4, 16, 64])
def test_search_coarse_matches_reference(pb, gi, built, nprobe):
    ix, _ = built
    for tau in (20, 26, 64):
        for cap in (0, 1500):
            key = f"p{nprobe}_t{tau}_c{cap}"
            st = pb.SearchStats()
            ids, sc, cnt = ix.search(gi["queries"], pb.CoarseParams(pb.Strategy.dual, 50, tau, nprobe, cap), st)
            assert np.array_equal(ids, gi[key + "_ids"]), key
            assert np.array_equal(_bits(sc), _bits(gi[key + "_scores"])), key
            assert np.array_equal(cnt, gi[key + "_counts"]), key
            assert st.survivors == int(gi[key + "_surv"].sum()), key
            _, _, _, _, scanned, _ = oracle.ivf_search(gi["pq"], gi["coarse"], gi["lists"], gi["queries"], 50,
                                                       nprobe, tau=tau, cap=cap)
            assert st.scanned == int(scanned.sum()), key


def test_strategies_edges_and_codes_path(pb, gi, built):
    ix, _ = built
    for strat in ("adc", "binary"):
        ids, sc, cnt = ix.search(gi["queries"], pb.CoarseParams(pb.strategy_from_string(strat), 50, 0, 16, 0))
        assert np.array_equal(ids, gi[f"{strat}16_ids"])
        assert np.array_equal(_bits(sc), _bits(gi[f"{strat}16_scores"]))
    ids, sc, cnt = ix.search(gi["queries"][:3], pb.CoarseParams(pb.Strategy.dual, 0, 26, 4, 0))
    assert cnt.tolist() == [0, 0, 0]
    with pytest.raises(pb.PolyError):
        ix.search(gi["queries"][:3], pb.CoarseParams(pb.Strategy.dual, 10, 65, 4, 0))
    empty = _ivf(pb, gi)
    ids, sc, cnt = empty.search(gi["queries"][:3], pb.CoarseParams(pb.Strategy.dual, 10, 26, 4, 0))
    assert (cnt == 0).all() and (ids == -1).all()
    # serialization path: the golden lists re-added as codes give the golden answers
    ix2 = _ivf(pb, gi)
    cells = np.repeat(np.arange(64, dtype=np.uint32), np.diff(gi["off"]).astype(np.int64))
    ix2.add_codes(cells, gi["list_codes"], gi["list_ids"])
    ids, sc, cnt = ix2.search(gi["queries"], pb.CoarseParams(pb.Strategy.dual, 50, 26, 16, 1500))
    assert np.array_equal(ids, gi["p16_t26_c1500_ids"])


def test_larger_ivf_matches_oracle(pb, gi):
    """256 cells, 300k codes, 300 queries (two batches), several nprobe / tau."""
    seed = int(gi["data_seed"])
    centers = oracle.gen_centers(seed, 1000, 128)
    rng = np.random.default_rng(5)
    train = oracle.gen_points(seed, 1, 0, 20000, centers)
    coarse = train[rng.choice(20000, 256, replace=False)]
    base = oracle.gen_points(seed, 2, 0, 300_000, centers)
    pq = gi["pq"]
    lists, assign = oracle.ivf_build(pq, base, coarse)
    ix = pb.IVFIndex(pb.ProductQuantizer(8, 8, 128, gi["codebooks"], gi["perms"]), coarse)
    ix.add(base)
    assert np.array_equal(ix.assign(base[:5000]), assign[:5000])
    queries = oracle.gen_points(seed, 3, 0, 300, centers)
    for nprobe, tau, cap in ((8, 26, 0), (32, 24, 0), (32, 64, 0), (64, 28, 20000)):
        oi, osc, oc, osv, _, _ = oracle.ivf_search(pq, coarse, lists, queries, 100, nprobe, tau=tau, cap=cap,
                                                   threads=16)
        st = pb.SearchStats()
        ids, sc, cnt = ix.search(queries, pb.CoarseParams(pb.Strategy.dual, 100, tau, nprobe, cap), st)
        assert np.array_equal(ids, oi), (nprobe, tau, cap)
        assert np.array_equal(_bits(sc), _bits(osc))
        assert np.array_equal(cnt, oc)
        if tau < 64:
            assert st.survivors == int(osv.sum())


def test_knn_graph_matches_oracle(pb, gi):
    """knn_graph on unit-normalised 256-d data, m = 16 codes."""
    import torch
    seed = int(gi["data_seed"])
    centers = oracle.gen_centers(seed, 4096, 256)
    z = np.load(os.path.join(os.path.dirname(GOLDEN), "pq_d256_m16.npz"))
    pq = oracle.PQ(16, 8, 256, z["codebooks"], z["perms"])
    x = oracle.gen_points(seed, 2, 0, 30000, centers, normalize=True)
    coarse = oracle.gen_points(seed, 1, 0, 128, centers, normalize=True)
    lists, _ = oracle.ivf_build(pq, x, coarse)
    ix = pb.IVFIndex(pb.ProductQuantizer(16, 8, 256, z["codebooks"], z["perms"]), coarse)
    ix.add(x)
    nq, k = 3000, 10
    dx = torch.from_numpy(x[:nq]).cuda()
    ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    sc = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    ix.knn_graph_device(dx, 0, pb.CoarseParams(pb.Strategy.dual, k, 52, 8, 0), ids, sc, cnt)
    torch.cuda.synchronize()
    oi, osc, oc, _, _, _ = oracle.ivf_search(pq, coarse, lists, x[:nq], k + 1, 8, tau=52, threads=16)
    for i in range(nq):
        row, srow = list(oi[i, :oc[i]]), list(osc[i, :oc[i]])
        if i in row:
            j = row.index(i)
            del row[j], srow[j]
        row, srow = row[:k], srow[:k]
        got = ids[i].cpu().numpy()
        assert got[:len(row)].tolist() == row, i
        assert int(cnt[i]) == len(row)
        assert (got[len(row):] == -1).all()


def test_knn_graph_file_sink(pb, gi, tmp_path):
    """The k-NN graph output sink: rows written in two appends (small
    batches: several pipelined steps each) read back equal to knn_graph_device, the file is
    byte-identical to the reference writer's, and the ivecs export holds the same ids."""
    import torch
    from paper_1609_01882_b200 import knn_format
    seed = int(gi["data_seed"])
    centers = oracle.gen_centers(seed, 1000, 128)
    x = oracle.gen_points(seed, 2, 0, 20000, centers)
    coarse = oracle.gen_points(seed, 1, 0, 64, centers)
    ix = pb.IVFIndex(pb.ProductQuantizer(8, 8, 128, gi["codebooks"], gi["perms"]), coarse)
    ix.add(x)
    ix.set_batch(50)  # steps of 64 x 50 rows: the write pipeline runs several steps per call
    n, k = 7000, 5
    p = pb.CoarseParams(pb.Strategy.dual, k, 26, 4, 0)
    dx = torch.from_numpy(x[:n]).cuda()
    ids = torch.empty((n, k), dtype=torch.int64, device="cuda")
    sc = torch.empty((n, k), dtype=torch.float32, device="cuda")
    cnt = torch.empty(n, dtype=torch.int32, device="cuda")
    ix.knn_graph_device(dx, 0, p, ids, sc, cnt)
    torch.cuda.synchronize()
    ids, sc, cnt = ids.cpu().numpy(), sc.cpu().numpy(), cnt.cpu().numpy().astype(np.uint32)
    path, vpath = tmp_path / "g.knng", tmp_path / "g.ivecs"
    with pb.KnnGraphWriter(path, k, vpath) as w:
        ix.knn_graph_write_device(w, dx[:4000], 0, p)
        ix.knn_graph_write_device(w, dx[4000:], 4000, p)
    assert w.records == n
    kk, rid, rc, rn, rs = knn_format.read_graph(path, check_sum=False)
    assert kk == k and np.array_equal(rid, np.arange(n)) and np.array_equal(rc, cnt)
    assert np.array_equal(rn, ids) and np.array_equal(_bits(rs), _bits(sc))
    ref = tmp_path / "ref.knng"
    knn_format.write_graph(ref, k, np.arange(500), cnt[:500], ids[:500], sc[:500])
    head = open(path, "rb").read()
    want = open(ref, "rb").read()
    assert head[48:len(want)] == want[48:]  # the first 500 records, byte for byte
    assert np.array_equal(knn_format.read_ivecs(vpath), ids.astype(np.int32))
    with pytest.raises(pb.PolyError):
        pb.KnnGraphWriter(tmp_path / "no_such_dir" / "g.knng", k)


@pytest.mark.parametrize("dim,nlist", [(128, 8192), (256, 4096)])
def test_probe_order_many_near_ties(pb, gi, dim, nlist):
    """enumerate_cells runs TF32 tensor-core dots + an exact re-rank (K5r): probe order
    must stay bit-exact, also with clustered cells (many near ties), exact duplicate
    cells (ties -> lower cell) and nprobe up to 1000, against the oracle's exact
    sq_l2 order."""
    seed = int(gi["data_seed"])
    centers = oracle.gen_centers(seed, 200, dim)  # 200 clusters: dozens of near-equidistant cells each
    coarse = oracle.gen_points(seed, 1, 0, nlist, centers)
    coarse[nlist // 2: nlist // 2 + 64] = coarse[:64]  # exact duplicates
    queries = oracle.gen_points(seed, 3, 0, 40, centers)
    queries[:4] = coarse[[3, 10, 70, nlist // 2 + 5]]  # queries sitting exactly on (duplicated) cells
    m = dim // 16
    zz = np.load(os.path.join(os.path.dirname(GOLDEN), "pq_d128_m8.npz" if dim == 128 else "pq_d256_m16.npz"))
    opq = oracle.PQ(m, 8, dim, zz["codebooks"], zz["perms"])
    empty = oracle.IVFLists(np.zeros(nlist + 1, np.uint64), np.zeros((0, m), np.uint8), np.zeros(0, np.int64))
    ix = pb.IVFIndex(pb.ProductQuantizer(m, 8, dim, zz["codebooks"], zz["perms"]), coarse)
    for nprobe in (1, 16, 100, 1000):
        want = oracle.ivf_search(opq, coarse, empty, queries, 1, nprobe, threads=16)[5]
        assert np.array_equal(ix.probes(queries, nprobe), want), nprobe


def test_by_list_sharding_matches_unsharded(pb, gi):
    """By-list sharding: 4 shards each holding whole lists (assign_lists
    by size), the same all-gathered probes, per-shard keys merged == the unsharded search;
    every shard only scans (and builds LUTs for) its own lists: scanned totals add up."""
    import torch
    from paper_1609_01882_b200.distributed import assign_lists, by_list_balance
    seed = int(gi["data_seed"])
    centers = oracle.gen_centers(seed, 1000, 128)
    rng = np.random.default_rng(12)
    coarse = oracle.gen_points(seed, 1, 0, 20000, centers)[rng.choice(20000, 256, replace=False)]
    n = 150_000
    base = oracle.gen_points(seed, 2, 0, n, centers)
    queries = oracle.gen_points(seed, 3, 0, 300, centers)
    mk = lambda: pb.IVFIndex(pb.ProductQuantizer(8, 8, 128, gi["codebooks"], gi["perms"]), coarse)  # noqa: E731
    full = mk()
    full.add(base)
    cells = full.assign(base)
    sizes = np.bincount(cells, minlength=256)
    owner = assign_lists(sizes, 4)
    loads = np.bincount(owner, weights=sizes, minlength=4)
    assert loads.max() - loads.min() <= sizes.max()  # LPT: within one list of each other
    shards = []
    for r in range(4):
        rows = np.nonzero(owner[cells] == r)[0]
        ix = mk()
        ix.add(base[rows], cells=cells[rows], ids=rows)
        shards.append(ix)
    k = 100
    dq = torch.from_numpy(queries).cuda()
    for nprobe, tau in ((8, 26), (32, 24), (32, 64)):
        p = pb.CoarseParams(pb.Strategy.dual, k, tau, nprobe, 0)
        want_ids, want_sc, want_cnt = full.search(queries, p)
        probes = torch.empty((300, nprobe), dtype=torch.int64, device="cuda")
        full.probe_keys_device(dq, nprobe, probes)
        keys = torch.empty((4, 300, k), dtype=torch.int64, device="cuda")
        cnts = torch.empty((4, 300), dtype=torch.int32, device="cuda")
        st = pb.SearchStats()
        for r, ix in enumerate(shards):
            ix.search_keys_device(dq, p, keys[r], cnts[r], stats=st, probes=probes)
        ids = torch.empty((300, k), dtype=torch.int64, device="cuda")
        sc = torch.empty((300, k), dtype=torch.float32, device="cuda")
        cnt = torch.empty(300, dtype=torch.int32, device="cuda")
        shards[0].merge_keys_device(keys, cnts, 4, 300, k, ids, sc, cnt)
        torch.cuda.synchronize()
        assert np.array_equal(ids.cpu().numpy(), want_ids), (nprobe, tau)
        assert np.array_equal(_bits(sc.cpu().numpy()), _bits(want_sc))
        assert np.array_equal(cnt.cpu().numpy(), want_cnt)
        st_full = pb.SearchStats()
        full.search(queries, p, st_full)
        assert st.scanned == st_full.scanned and st.survivors == st_full.survivors
        pc = (probes.cpu().numpy() & 0xFFFFFFFF).astype(np.int64)
        imb, per = by_list_balance(sizes, pc, owner, 4)
        assert per.sum() == st_full.scanned and imb >= 1.0
        # the two-phase protocol: round 1 on the owner of each first probe, bounds min-reduced,
        # round 2 everywhere under the global bound -- same merged result, fewer candidates
        thr = torch.empty((4, 300), dtype=torch.int64, device="cuda")
        for r, ix in enumerate(shards):
            ix.search_keys_phase_device(dq, p, probes, 1, thr[r])
        none = torch.full_like(thr[0], 2**63 - 1)
        g = torch.where(thr == -1, none, thr).min(0).values
        g = torch.where(g == 2**63 - 1, torch.full_like(g, -1), g)
        st2 = pb.SearchStats()
        for r, ix in enumerate(shards):
            ix.search_keys_phase_device(dq, p, probes, 2, g.clone(), keys[r], cnts[r], stats=st2)
        shards[0].merge_keys_device(keys, cnts, 4, 300, k, ids, sc, cnt)
        torch.cuda.synchronize()
        assert np.array_equal(ids.cpu().numpy(), want_ids), ("2-phase", nprobe, tau)
        assert np.array_equal(_bits(sc.cpu().numpy()), _bits(want_sc))
        assert np.array_equal(cnt.cpu().numpy(), want_cnt)
        assert st2.scanned == st_full.scanned
    # the engine's by-list path at world size 1 (no process group: no reduce)
    from paper_1609_01882_b200.distributed import IVFIndexEngine, ShardedSearch
    p = pb.CoarseParams(pb.Strategy.dual, k, 26, 16, 0)
    want_ids, want_sc, want_cnt = full.search(queries, p)
    full.set_batch(128)  # several phase batches
    ids, sc, cnt = ShardedSearch(IVFIndexEngine(full, by_list=True)).search_batch(dq, p)
    torch.cuda.synchronize()
    assert np.array_equal(ids.cpu().numpy(), want_ids) and np.array_equal(cnt.cpu().numpy(), want_cnt)
    with pytest.raises(pb.PolyError):  # phase 2 without phase 1
        shards[1].search_keys_phase_device(dq, p, probes[:, :16].contiguous(), 2, g.clone(), keys[1], cnts[1])


def test_sharded_ivf_merge_matches_unsharded(pb, gi):
    """SURVEY.md sec. 8e for IVF: 4 shards (every cell's list restricted to an id range),
    per-shard top-k keys, exact K3 merge == the unsharded search == the oracle; the
    NCCL world-1 path of ShardedSearch with the IVF engine gives the same."""
    import torch
    import torch.distributed as dist
    from paper_1609_01882_b200.distributed import IVFIndexEngine, ShardedSearch, shard_range
    seed = int(gi["data_seed"])
    centers = oracle.gen_centers(seed, 1000, 128)
    rng = np.random.default_rng(9)
    coarse = oracle.gen_points(seed, 1, 0, 20000, centers)[rng.choice(20000, 256, replace=False)]
    n = 200_000
    base = oracle.gen_points(seed, 2, 0, n, centers)
    queries = oracle.gen_points(seed, 3, 0, 300, centers)
    mk = lambda: pb.IVFIndex(pb.ProductQuantizer(8, 8, 128, gi["codebooks"], gi["perms"]), coarse)  # noqa: E731
    full = mk()
    full.add(base)
    shards = []
    for r in range(4):
        r0, r1 = shard_range(n, 4, r)
        ix = mk()
        ix.add(base[r0:r1], ids=np.arange(r0, r1))
        shards.append(ix)
    k = 100
    dq = torch.from_numpy(queries).cuda()
    for nprobe, tau in ((8, 26), (32, 64)):
        p = pb.CoarseParams(pb.Strategy.dual, k, tau, nprobe, 0)
        want_ids, want_sc, want_cnt = full.search(queries, p)
        keys = torch.empty((4, 300, k), dtype=torch.int64, device="cuda")
        cnts = torch.empty((4, 300), dtype=torch.int32, device="cuda")
        st = pb.SearchStats()
        for r, ix in enumerate(shards):
            ix.search_keys_device(dq, p, keys[r], cnts[r], stats=st)
        ids = torch.empty((300, k), dtype=torch.int64, device="cuda")
        sc = torch.empty((300, k), dtype=torch.float32, device="cuda")
        cnt = torch.empty(300, dtype=torch.int32, device="cuda")
        shards[0].merge_keys_device(keys, cnts, 4, 300, k, ids, sc, cnt)
        torch.cuda.synchronize()
        assert np.array_equal(ids.cpu().numpy(), want_ids), (nprobe, tau)
        assert np.array_equal(_bits(sc.cpu().numpy()), _bits(want_sc))
        assert np.array_equal(cnt.cpu().numpy(), want_cnt)
        st_full = pb.SearchStats()
        full.search(queries, p, st_full)
        assert st.scanned == st_full.scanned and st.survivors == st_full.survivors
    # the same through the rank plumbing, world = 1 over NCCL
    if not dist.is_initialized():
        import os as _os
        _os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        _os.environ.setdefault("MASTER_PORT", "29631")
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        p = pb.CoarseParams(pb.Strategy.dual, k, 26, 8, 0)
        want_ids, _, _ = full.search(queries, p)
        for split in (False, True):  # split: coarse quantization by query slice + all-gather of probes
            ids, sc, cnt = ShardedSearch(IVFIndexEngine(full, split_coarse=split)).search_batch(dq, p)
            torch.cuda.synchronize()
            assert np.array_equal(ids.cpu().numpy(), want_ids), split
    finally:
        dist.destroy_process_group()
    # probes enumerated in query slices (as two ranks would) and passed in == enumerated inside
    p = pb.CoarseParams(pb.Strategy.dual, k, 26, 8, 0)
    pr = torch.empty((300, 8), dtype=torch.int64, device="cuda")
    shards[1].probe_keys_device(dq[:170], 8, pr[:170])
    shards[1].probe_keys_device(dq[170:], 8, pr[170:])
    ref = torch.empty((300, 8), dtype=torch.int64, device="cuda")
    shards[1].probe_keys_device(dq, 8, ref)
    torch.cuda.synchronize()
    assert torch.equal(pr, ref)
    assert np.array_equal((ref.cpu().numpy() & 0xFFFFFFFF).astype(np.uint32), full.probes(queries, 8))
    for r, ix in enumerate(shards):
        k_in = torch.empty((300, k), dtype=torch.int64, device="cuda")
        c_in = torch.empty(300, dtype=torch.int32, device="cuda")
        ix.search_keys_device(dq, p, keys[r], cnts[r])
        ix.search_keys_device(dq, p, k_in, c_in, probes=pr)
        torch.cuda.synchronize()
        assert torch.equal(k_in, keys[r]) and torch.equal(c_in, cnts[r]), r
    # ids outside [0, 2^32) need a rank table, whose ranks are shard-local: rejected
    odd = mk()
    odd.add(base[:1000], ids=np.arange(1000) * 3 + 2**33)
    with pytest.raises(pb.PolyError) as e:
        odd.search_keys_device(dq, pb.CoarseParams(pb.Strategy.dual, k, 26, 8, 0), keys[0], cnts[0])
    assert e.value.code == pb.Errc.state
    # scattered ids below 2^32 ride in the key (by-list shards hold such ids)
    sc3 = mk()
    sc3.add(base[:1000], ids=np.arange(1000) * 3)
    sc3.search_keys_device(dq, pb.CoarseParams(pb.Strategy.dual, k, 26, 8, 0), keys[0], cnts[0])
    torch.cuda.synchronize()
    got = keys[0].cpu().numpy()
    ok = got != -1
    assert ok.any() and (((got[ok] & 0xFFFFFFFF) % 3) == 0).all()


def test_full_config2_size(pb):
    """BASELINE config 2 at its per-GPU size: 1.25e8 residual codes in 65,536 lists (the
    bench's build: GPU generator, TF32 nearest-cell assignment, exact residual encoding).
    The oracle searches the identical lists (read back with lists()): 4 queries exact at
    nprobe 16; every returned neighbour of a 256-query batch lies in one of its query's
    probed cells."""
    import time
    import torch
    from paper_1609_01882_b200 import synth
    seed = 160901882
    z = np.load(os.path.join(os.path.dirname(GOLDEN), "pq_ivf65536_d128_m8.npz"))
    pq = pb.ProductQuantizer(8, 8, 128, z["codebooks"], z["perms"])
    opq = oracle.PQ(8, 8, 128, z["codebooks"], z["perms"])
    centers = synth.gen_centers(seed, 1000, 128)
    coarse = synth.gen_points(seed, 1, 0, 65536, centers)
    ivf = pb.IVFIndex(pq, coarse)
    n, chunk = 125_000_000, 1 << 22
    t = time.time()
    torch.backends.cuda.matmul.allow_tf32 = True
    dc = torch.from_numpy(coarse).cuda()
    cn = (dc * dc).sum(1)
    x = torch.empty((chunk, 128), device="cuda")
    cells = torch.empty(chunk, dtype=torch.int32, device="cuda")
    for r in range(0, n, chunk):
        nb = min(chunk, n - r)
        pb.gen_points_device(centers, seed, 2, r, nb, x[:nb])
        for b in range(0, nb, 16384):
            xs = x[b:min(b + 16384, nb)]
            cells[b:b + xs.shape[0]] = torch.argmin(cn[None, :] - 2.0 * (xs @ dc.T), dim=1).to(torch.int32)
        ivf.add_device(x[:nb], cells[:nb], r)
    torch.cuda.synchronize()
    build_s = time.time() - t
    queries = synth.gen_points(seed, 3, 0, 256, centers)
    p = pb.CoarseParams(pb.Strategy.dual, 100, 26, 16, 0)
    ids, sc, cnt = ivf.search(queries, p)
    off, codes, lids = ivf.lists()
    lists = oracle.IVFLists(off, codes, lids)
    sub = np.array([0, 85, 170, 255])
    oi, osc, oc, _, _, pr = oracle.ivf_search(opq, coarse, lists, queries[sub], 100, 16, tau=26,
                                              threads=os.cpu_count() or 8)
    assert _same(ids[sub], oi)
    assert _same(_bits(sc[sub]), _bits(osc))
    assert _same(cnt[sub], oc)
    assert _same(ivf.probes(queries[sub], 16), pr)
    # every returned neighbour sits in one of its query's probed cells
    probes = ivf.probes(queries, 16)
    cell_of = np.empty(n, np.int64)
    cell_of[lids] = np.repeat(np.arange(65536), np.diff(off).astype(np.int64))
    for qi in range(256):
        got = ids[qi, :cnt[qi]]
        assert np.isin(cell_of[got], probes[qi]).all(), qi
    print(f"build {build_s:.1f} s")


def _same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


def test_full_config4_size(pb):
    """BASELINE config 4 at its full size: 1e7 unit-normalised 256-d vectors, IVF 16,384
    + PQ m=16, knn_graph with nprobe 32, ht 52, k 10 for 2,048 rows;
    4 rows exact against the oracle on the same lists (k + 1 results, self removed)."""
    import torch
    from paper_1609_01882_b200 import synth
    seed = 160901882
    z = np.load(os.path.join(os.path.dirname(GOLDEN), "pq_ivf16384_d256_m16.npz"))
    pq = pb.ProductQuantizer(16, 8, 256, z["codebooks"], z["perms"])
    opq = oracle.PQ(16, 8, 256, z["codebooks"], z["perms"])
    centers = synth.gen_centers(seed, 4096, 256)
    coarse = synth.gen_points(seed, 1, 0, 16384, centers, normalize=True)
    ivf = pb.IVFIndex(pq, coarse)
    n, chunk = 10_000_000, 1 << 21
    torch.backends.cuda.matmul.allow_tf32 = True
    dc = torch.from_numpy(coarse).cuda()
    cn = (dc * dc).sum(1)
    x = torch.empty((chunk, 256), device="cuda")
    cells = torch.empty(chunk, dtype=torch.int32, device="cuda")
    for r in range(0, n, chunk):
        nb = min(chunk, n - r)
        pb.gen_points_device(centers, seed, 2, r, nb, x[:nb], normalize=True)
        for b in range(0, nb, 16384):
            xs = x[b:min(b + 16384, nb)]
            cells[b:b + xs.shape[0]] = torch.argmin(cn[None, :] - 2.0 * (xs @ dc.T), dim=1).to(torch.int32)
        ivf.add_device(x[:nb], cells[:nb], r)
    row0, rows, k = 4_000_000, 2048, 10
    dx = torch.empty((rows, 256), device="cuda")
    pb.gen_points_device(centers, seed, 2, row0, rows, dx, normalize=True)
    ids = torch.empty((rows, k), dtype=torch.int64, device="cuda")
    sc = torch.empty((rows, k), dtype=torch.float32, device="cuda")
    cnt = torch.empty(rows, dtype=torch.int32, device="cuda")
    ivf.knn_graph_device(dx, row0, pb.CoarseParams(pb.Strategy.dual, k, 52, 32, 0), ids, sc, cnt)
    torch.cuda.synchronize()
    off, codes, lids = ivf.lists()
    lists = oracle.IVFLists(off, codes, lids)
    sub = np.array([0, 700, 1400, 2047])
    xq = dx[sub].cpu().numpy()
    oi, osc, oc, _, _, _ = oracle.ivf_search(opq, coarse, lists, xq, k + 1, 32, tau=52, threads=os.cpu_count() or 8)
    for j, r in enumerate(sub):
        row, srow = list(oi[j, :oc[j]]), list(osc[j, :oc[j]])
        if row0 + r in row:
            i = row.index(row0 + r)
            del row[i], srow[i]
        row, srow = row[:k], srow[:k]
        assert ids[r].cpu().numpy()[:len(row)].tolist() == row, r
        assert _same(_bits(sc[r].cpu().numpy()[:len(row)]), _bits(np.array(srow, np.float32)))
        assert int(cnt[r]) == len(row)


@pytest.mark.parametrize("seed", range(20))
def test_randomized_ivf_against_oracle(pb, gi, seed):
    """Randomised IVF sweep (cells, list sizes, nprobe incl. > 64, cap, tau, strategy, k,
    ids) of search_coarse against the oracle (exact assignment + residual encoding on
    both sides, so the lists are the same)."""
    rng = np.random.default_rng(2000 + seed)
    dseed = int(gi["data_seed"])
    centers = oracle.gen_centers(dseed, 1000, 128)
    nlist = int(rng.choice([1, 3, 64, 200, 1024]))
    n = int(rng.choice([0, 1, 500, 5000, 40000]))
    coarse = oracle.gen_points(dseed, 1, int(rng.integers(0, 1000)), nlist, centers)
    base = oracle.gen_points(dseed, 2, int(rng.integers(0, 10_000)), n, centers) if n else np.zeros((0, 128), np.float32)
    ids = (rng.permutation(n).astype(np.int64) * 5 + 1) if seed % 2 else np.arange(n, dtype=np.int64)
    nq = int(rng.choice([1, 17, 256, 300, 2100]))  # 2100: more than one 2048-query batch
    queries = oracle.gen_points(dseed, 3, int(rng.integers(0, 1000)), nq, centers)
    nprobe = int(min(nlist, rng.choice([1, 4, 16, 65, 100])))
    k = int(rng.choice([1, 10, 100]))
    strategy = ["dual", "dual", "adc", "binary", "disidx"][seed % 5]
    tau = int(rng.integers(0, 65)) if strategy == "dual" else 64
    cap = int(rng.choice([0, 0, 300]))
    batch = int(rng.choice([7, 64, 5000])) if seed % 4 == 3 else None  # queries per internal batch
    pq = gi["pq"]
    ix = pb.IVFIndex(pb.ProductQuantizer(8, 8, 128, gi["codebooks"], gi["perms"]), coarse)
    if batch:
        ix.set_batch(batch)
        assert ix.batch == batch
    if n:
        ix.add(base, ids=ids)
        lists, _ = oracle.ivf_build(pq, base, coarse, ids=ids)
    else:
        lists = oracle.IVFLists(np.zeros(nlist + 1, np.uint64), np.zeros((0, 8), np.uint8), np.zeros(0, np.int64))
    oi, osc, oc, osv, oscan, opr, osh = oracle.ivf_search(pq, coarse, lists, queries, k, nprobe, tau=tau,
                                                          strategy=strategy, cap=cap, threads=16, return_hash=True)
    st = pb.SearchStats()
    gi_, gsc, gc = ix.search(queries, pb.CoarseParams(pb.strategy_from_string(strategy), k, tau, nprobe, cap), st)
    if n and strategy == "dual":  # per-query survivor sets (count + id hash) through the device API
        import torch
        dq = torch.from_numpy(queries).cuda()
        d = [torch.empty((nq, k), dtype=torch.int64, device="cuda"), torch.empty((nq, k), dtype=torch.float32,
                                                                                 device="cuda")]
        sv = torch.empty(nq, dtype=torch.int64, device="cuda")
        sh = torch.empty(nq, dtype=torch.int64, device="cuda")
        ix.search_device(dq, pb.CoarseParams(pb.Strategy.dual, k, tau, nprobe, cap), d[0], d[1],
                         stream=torch.cuda.current_stream().cuda_stream, d_survivors=sv, d_survivor_hash=sh)
        torch.cuda.synchronize()
        assert np.array_equal(sv.cpu().numpy().view(np.uint64), osv), (nlist, n, nq, nprobe, k, tau, cap)
        assert np.array_equal(sh.cpu().numpy().view(np.uint64), osh), (nlist, n, nq, nprobe, k, tau, cap)
        assert np.array_equal(d[0].cpu().numpy(), oi)
    ctx = (nlist, n, nq, nprobe, k, strategy, tau, cap, batch)
    assert np.array_equal(ix.probes(queries, nprobe), opr), ctx
    assert np.array_equal(gi_, oi), ctx
    assert np.array_equal(_bits(gsc), _bits(osc)), ctx
    assert np.array_equal(gc, oc), ctx
    if n and strategy == "dual" and tau < 64:
        assert st.survivors == int(osv.sum()), ctx
