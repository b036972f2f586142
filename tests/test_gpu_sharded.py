"""GPU parity of the single-process multi-GPU FlatIndex (poly_b200_sharded_*, SURVEY.md
sec. 8(b)): the shards (several on one GPU here: the pool has one B200 per box) merged
on devices[0] give exactly the single-index answers and the reference goldens -- ids
(ties included), score bits, counts and the summed statistics."""
import os
import subprocess

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1609_01882_b200 as pb
    return pb


def _bits(x):
    return np.ascontiguousarray(x, np.float32).view(np.uint32)


def _pq(pb, pq):
    return pb.ProductQuantizer(pq.m, pq.dbits, pq.dim, pq.codebooks, pq.perms)


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
def test_sharded_matches_goldens(pb, pq8, g8, shards):
    sx = pb.ShardedFlatIndex(_pq(pb, pq8), [0] * shards)
    sx.add_codes(g8["codes"])
    assert sx.size() == len(g8["codes"])
    assert sum(sx.shard_sizes()) == len(g8["codes"])
    for tau in (20, 24, 28, 32, 64):
        st = pb.SearchStats()
        ids, sc, cnt = sx.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.dual, 100, tau), st)
        key = f"dual{tau}"
        assert np.array_equal(ids, g8[key + "_ids"]), (shards, tau)
        assert np.array_equal(_bits(sc), _bits(g8[key + "_scores"])), (shards, tau)
        assert np.array_equal(cnt, g8[key + "_counts"]), (shards, tau)
        assert st.scanned == len(g8["codes"]) * len(g8["queries"])
        if tau < 64:
            assert st.survivors == int(g8[key + "_surv"].sum()), (shards, tau)


@pytest.mark.parametrize("strategy", ["dual", "adc", "binary", "disidx"])
def test_sharded_equals_single_index(pb, pq8, strategy):
    """200k synthetic codes with permuted ids (each shard maps ids through a rank table),
    three add calls, 5 shards: equal to one FlatIndex, and to the oracle on 8 queries."""
    seed = 160901882
    centers = oracle.gen_centers(seed, 1000, 128)
    one = pb.FlatIndex(_pq(pb, pq8))
    one.add_synthetic(seed, centers, 0, 200_000)
    codes = one.codes()
    ids = np.random.default_rng(7).permutation(200_000).astype(np.int64) * 11 - 50_000
    ref = pb.FlatIndex(_pq(pb, pq8))
    ref.add_codes(codes, ids)
    sx = pb.ShardedFlatIndex(_pq(pb, pq8), [0] * 5)
    for a, b in ((0, 1000), (1000, 150_001), (150_001, 200_000)):
        sx.add_codes(codes[a:b], ids[a:b])
    q = oracle.gen_points(seed, 3, 0, 300, centers)
    s = pb.strategy_from_string(strategy)
    for tau, k in ((24, 100), (28, 1), (16, 2048)):
        p = pb.SearchParams(s, k, tau if strategy == "dual" else 64)
        st1, st2 = pb.SearchStats(), pb.SearchStats()
        i1, s1, c1 = ref.search_batch(q, p, st1)
        i2, s2, c2 = sx.search_batch(q, p, st2)
        assert np.array_equal(i1, i2) and np.array_equal(_bits(s1), _bits(s2)) and np.array_equal(c1, c2), (tau, k)
        assert (st1.scanned, st1.survivors) == (st2.scanned, st2.survivors)
        oi, osc, oc, _, _ = oracle.search(pq8, codes, q[:8], p.k, p.tau, strategy=strategy, ids=ids, threads=16)
        assert np.array_equal(i2[:8], oi) and np.array_equal(_bits(s2[:8]), _bits(osc)), (tau, k)


def test_sharded_edges(pb, pq8, g8):
    sx = pb.ShardedFlatIndex(_pq(pb, pq8), [0, 0])
    ids, sc, cnt = sx.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.dual, 10, 24))  # empty index
    assert (cnt == 0).all() and (ids == -1).all() and np.isinf(sc).all()
    sx.add_codes(g8["codes"][:3])  # the two shards get 1 and 2 rows
    ids, sc, cnt = sx.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.adc, 10, 64))
    assert (cnt == 3).all() and (ids[:, 3:] == -1).all()
    ids, sc, cnt = sx.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.adc, 0, 64))
    assert ids.shape == (len(g8["queries"]), 0) and (cnt == 0).all()
    with pytest.raises(pb.PolyError) as e:
        sx.search_batch(g8["queries"], pb.SearchParams(pb.Strategy.dual, 10, 65))
    assert e.value.code == pb.Errc.invalid_argument
    with pytest.raises(pb.PolyError):
        pb.ShardedFlatIndex(_pq(pb, pq8), [])


def test_cpp_sharded_mirror(pb, pq8, g8, tmp_path):
    """A C++ caller of poly_b200::ShardedFlatIndex gets the reference's answers."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_1609_01882_b200")
    exe = str(tmp_path / "sharded")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "sharded_smoke.cpp"), "-L", libdir, "-lpoly_b200",
                    f"-Wl,-rpath,{libdir}", "-lpthread", "-o", exe], check=True)
    cb, pm, blob = (str(tmp_path / f) for f in ("cb.bin", "perms.bin", "blob.bin"))
    pq8.codebooks.tofile(cb)
    pq8.perms.tofile(pm)
    with open(blob, "wb") as f:
        f.write(g8["codes"].tobytes())
        f.write(g8["queries"].astype(np.float32).tobytes())
    out = subprocess.run([exe, cb, pm, blob, "4"], capture_output=True, text=True, check=True).stdout.split("\n")
    assert out[0] == f"stats {20000 * 24} {int(g8['dual24_surv'].sum())}"
    for i in range(24):
        assert [int(x) for x in out[1 + i].split()] == g8["dual24_ids"][i, :10].tolist()
    assert out[25] == "error 1"
