"""Survivor-set parity and the candidate-list overflow path, through the C ABI.

North star: "bit-exact for Hamming distances, survivor sets and ... top-k ids"
(SearchStats.survivors flat_index.hpp:54-57).  The GPU
reports, per query, the number of codes that pass the dual filter and an
order-independent hash of that set (sum of mix64(id) mod 2^64); the oracle
computes the same over its pass-1 survivor list (oracle/polyoracle.c).  Equal
counts and hashes per query pin the survivor set itself, not just its size.

The overflow tests drive the exact rescue scan (csrc/kernels_rescue.cu): a
database ordered so that keys arrive in descending order (the worst case for
the running-bound candidate lists), and a forced small list capacity.
"""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
THREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def pb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1609_01882_b200 as pb
    return pb


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def _pbpq(pb, pq):
    return pb.ProductQuantizer(pq.m, pq.dbits, pq.dim, pq.codebooks, pq.perms)


def _flat_dev(pb, ix, queries, params):
    """search_batch_device_ex: ids, scores, counts, per-query survivors and hashes."""
    import torch
    nq, k = len(queries), int(params.k)
    dq = torch.from_numpy(np.ascontiguousarray(queries, np.float32)).cuda()
    ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    sc = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    sv = torch.empty(nq, dtype=torch.int64, device="cuda")
    sh = torch.empty(nq, dtype=torch.int64, device="cuda")
    ix.search_batch_device(dq, params, ids, sc, cnt, sv, stream=torch.cuda.current_stream().cuda_stream,
                           d_survivor_hash=sh)
    torch.cuda.synchronize()
    return (ids.cpu().numpy(), sc.cpu().numpy(), cnt.cpu().numpy().astype(np.uint32),
            sv.cpu().numpy().view(np.uint64), sh.cpu().numpy().view(np.uint64))


@pytest.fixture(scope="module")
def big8(pb):
    z = np.load(os.path.join(GOLDEN, "pq_d128_m8.npz"))
    pq = oracle.PQ(8, 8, 128, z["codebooks"], z["perms"])
    seed = int(z["data_seed"])
    centers = oracle.gen_centers(seed, 1000, 128)
    ix = pb.FlatIndex(_pbpq(pb, pq))
    ix.add_synthetic(seed, centers, 0, 1_000_000)
    return pq, ix, ix.codes(), oracle.gen_points(seed, 3, 0, 300, centers), centers, seed


@pytest.mark.parametrize("tau", [0, 20, 24, 28, 32, 64])
def test_survivor_sets_million_codes(pb, big8, tau):
    """1M codes, 300 queries (two batches): per-query survivor count and survivor-set hash
    equal the oracle's pass-1 set, and the top-k is exact.  tau = 64 = code_bits: every
    code survives (dual == adc id-for-id)."""
    pq, ix, codes, queries, _, _ = big8
    oi, osc, oc, osv, osh = oracle.search(pq, codes, queries, 100, tau=tau, threads=THREADS)
    gi, gsc, gc, gsv, gsh = _flat_dev(pb, ix, queries, pb.SearchParams(pb.Strategy.dual, 100, tau))
    assert np.array_equal(gsv, osv), tau
    assert np.array_equal(gsh, osh), tau
    assert np.array_equal(gi, oi) and np.array_equal(_bits(gsc), _bits(osc)) and np.array_equal(gc, oc)


@pytest.mark.parametrize("seed", range(12))
def test_survivor_sets_randomized(pb, seed):
    """Random sizes, m = 8 / 16, taus, ids (positions, arbitrary < 2^32, offset): survivor
    counts and hashes per query equal the oracle's."""
    rng = np.random.default_rng(7000 + seed)
    wide = seed % 3 == 2
    name, gname = ("pq_d256_m16.npz", "golden_m16.npz") if wide else ("pq_d128_m8.npz", "golden_m8.npz")
    z = np.load(os.path.join(GOLDEN, name))
    pq = oracle.PQ(int(z["m"]), 8, int(z["dim"]), z["codebooks"], z["perms"])
    g = np.load(os.path.join(GOLDEN, gname))
    n = int(rng.choice([1, 255, 1537, 20000, 70000, 200000]))
    nq = int(rng.choice([1, 16, 17, 100, 257]))
    tau = int(rng.integers(0, pq.code_bits + 1))
    codes = g["codes"][rng.integers(0, g["codes"].shape[0], n)]
    ids = [None, rng.permutation(n).astype(np.int64) * 3 + 11, np.arange(n, dtype=np.int64) + 123456][seed % 3]
    queries = g["queries"][rng.integers(0, g["queries"].shape[0], nq)]
    ix = pb.FlatIndex(_pbpq(pb, pq))
    ix.add_codes(codes, ids)
    oids = np.arange(n, dtype=np.int64) if ids is None else ids
    oi, osc, oc, osv, osh = oracle.search(pq, codes, queries, 50, tau=tau, ids=oids, threads=THREADS)
    gi, gsc, gc, gsv, gsh = _flat_dev(pb, ix, queries, pb.SearchParams(pb.Strategy.dual, 50, tau))
    ctx = (n, nq, tau, wide, seed % 3)
    assert np.array_equal(gsv, osv), ctx
    assert np.array_equal(gsh, osh), ctx
    assert np.array_equal(gi, oi), ctx
    assert np.array_equal(_bits(gsc), _bits(osc)), ctx


@pytest.mark.parametrize("strategy,tau,k,expect", [("dual", 24, 100, False), ("dual", 32, 257, True),
                                                   ("adc", 64, 100, True), ("binary", 0, 100, True),
                                                   ("disidx", 0, 10, False)])
def test_forced_overflow_is_rescued_exactly(pb, big8, strategy, tau, k, expect):
    """With the candidate list shrunk to ~1-2 select blocks, queries overflow (where the
    seeded bound leaves more candidates than that: `expect`); the rescue scan must still
    return the oracle's exact top-k (ties included)."""
    pq, _, codes, queries, _, _ = big8
    sub = codes[:200_000]
    ix = pb.FlatIndex(_pbpq(pb, pq))
    ix.add_codes(sub)
    ix.debug_set_list_capacity(1024)
    q = queries[:40]
    oi, osc, oc, _, _ = oracle.search(pq, sub, q, k, tau=tau, strategy=strategy, threads=THREADS)
    gi, gsc, gc = ix.search_batch(q, pb.SearchParams(pb.strategy_from_string(strategy), k, tau))
    if expect:
        assert ix.debug_rescued() > 0, "the forced capacity should have overflowed"
    assert np.array_equal(gi, oi)
    assert np.array_equal(_bits(gsc), _bits(osc))
    assert np.array_equal(gc, oc)


def test_adversarial_descending_order(pb, big8):
    """A database sorted by descending ADC to query 0 (keys arrive in falling order, so the
    running bound never prunes and the default-size list overflows): exact results for
    query 0 and its neighbours, under the dual filter (k = 1000) and plain ADC (k = 2048)."""
    pq, _, _, queries, centers, seed = big8
    n = 20_000_000
    gen = pb.FlatIndex(_pbpq(pb, pq))
    gen.add_synthetic(seed, centers, 0, n)
    codes = gen.codes()
    del gen
    _, lutp, _ = oracle.lut_batch(pq, queries[:1])
    acc = lutp[0, 0][codes[:, 0]].astype(np.float32)
    for s in range(1, 8):  # adc_distance in sq order (pq.cpp:121-128)
        acc = (acc + lutp[0, s][codes[:, s]]).astype(np.float32)
    order = np.argsort(-acc, kind="stable")
    codes = np.ascontiguousarray(codes[order])
    ids = order.astype(np.int64)
    ix = pb.FlatIndex(_pbpq(pb, pq))
    ix.add_codes(codes, ids)
    q = queries[:8]
    for strategy, tau, k in (("dual", 24, 1000), ("adc", 64, 2048)):
        oi, osc, oc, _, _ = oracle.search(pq, codes, q, k, tau=tau, strategy=strategy, ids=ids, threads=THREADS)
        gi, gsc, gc = ix.search_batch(q, pb.SearchParams(pb.strategy_from_string(strategy), k, tau))
        assert ix.debug_rescued() >= 1, (strategy, "query 0 should overflow the default list")
        assert np.array_equal(gi, oi), strategy
        assert np.array_equal(_bits(gsc), _bits(osc)), strategy
        assert np.array_equal(gc, oc), strategy


# ---------------------------------------------------------------------------- IVF
@pytest.fixture(scope="module")
def gi():
    z = dict(np.load(os.path.join(GOLDEN, "golden_ivf.npz")))
    z["pq"] = oracle.PQ(8, 8, 128, z["codebooks"], z["perms"])
    return z


def _ivf_dev(pb, ix, queries, params):
    import torch
    nq, k = len(queries), int(params.k)
    dq = torch.from_numpy(np.ascontiguousarray(queries, np.float32)).cuda()
    ids = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    sc = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    sv = torch.empty(nq, dtype=torch.int64, device="cuda")
    sh = torch.empty(nq, dtype=torch.int64, device="cuda")
    ix.search_device(dq, params, ids, sc, cnt, stream=torch.cuda.current_stream().cuda_stream, d_survivors=sv,
                     d_survivor_hash=sh)
    torch.cuda.synchronize()
    return (ids.cpu().numpy(), sc.cpu().numpy(), cnt.cpu().numpy().astype(np.uint32),
            sv.cpu().numpy().view(np.uint64), sh.cpu().numpy().view(np.uint64))


@pytest.mark.parametrize("seed", range(8))
def test_ivf_survivor_sets_and_forced_overflow(pb, gi, seed):
    """IVF search_coarse: per-query survivor counts and hashes equal the oracle's; on odd
    seeds the candidate list is shrunk so that queries overflow and are rescued exactly."""
    rng = np.random.default_rng(9100 + seed)
    dseed = int(gi["data_seed"])
    centers = oracle.gen_centers(dseed, 1000, 128)
    nlist = int(rng.choice([16, 64, 256]))
    n = int(rng.choice([20000, 60000]))
    coarse = oracle.gen_points(dseed, 1, int(rng.integers(0, 1000)), nlist, centers)
    base = oracle.gen_points(dseed, 2, int(rng.integers(0, 10_000)), n, centers)
    ids = rng.permutation(n).astype(np.int64) * 5 + 1
    nq = int(rng.choice([17, 300]))
    queries = oracle.gen_points(dseed, 3, int(rng.integers(0, 1000)), nq, centers)
    nprobe = int(min(nlist, rng.choice([4, 16, 40])))
    k = int(rng.choice([10, 100]))
    tau = int(rng.choice([20, 26, 32, 64])) if seed % 2 == 0 else int(rng.choice([32, 64]))
    pq = gi["pq"]
    ix = pb.IVFIndex(pb.ProductQuantizer(8, 8, 128, gi["codebooks"], gi["perms"]), coarse)
    ix.add(base, ids=ids)
    if seed % 2:  # the list holds only k keys: round 1 alone overflows it
        ix.debug_set_list_capacity(k)
    lists, _ = oracle.ivf_build(pq, base, coarse, ids=ids)
    oi, osc, oc, osv, _, _, osh = oracle.ivf_search(pq, coarse, lists, queries, k, nprobe, tau=tau, threads=THREADS,
                                                    return_hash=True)
    gi_, gsc, gc, gsv, gsh = _ivf_dev(pb, ix, queries, pb.CoarseParams(pb.Strategy.dual, k, tau, nprobe, 0))
    ctx = (nlist, n, nq, nprobe, k, tau, seed % 2)
    if seed % 2:
        assert ix.debug_rescued() > 0, ctx
    assert np.array_equal(gsv, osv), ctx
    assert np.array_equal(gsh, osh), ctx
    assert np.array_equal(gi_, oi), ctx
    assert np.array_equal(_bits(gsc), _bits(osc)), ctx
    assert np.array_equal(gc, oc), ctx


def test_ivf_nprobe_above_limit_is_rejected(pb, gi):
    """min(nprobe, nlist) > 2048 is rejected (invalid_argument), not run past the K3 buffers."""
    dseed = int(gi["data_seed"])
    centers = oracle.gen_centers(dseed, 1000, 128)
    coarse = oracle.gen_points(dseed, 1, 0, 4096, centers)
    ix = pb.IVFIndex(pb.ProductQuantizer(8, 8, 128, gi["codebooks"], gi["perms"]), coarse)
    ix.add(oracle.gen_points(dseed, 2, 0, 5000, centers))
    q = oracle.gen_points(dseed, 3, 0, 4, centers)
    with pytest.raises(pb.PolyError) as e:
        ix.search(q, pb.CoarseParams(pb.Strategy.dual, 10, 24, 4096, 0))
    assert e.value.code == pb.Errc.invalid_argument
    ids, _, _ = ix.search(q, pb.CoarseParams(pb.Strategy.dual, 10, 24, 2048, 0))  # the limit itself runs
    assert ids.shape == (4, 10)
