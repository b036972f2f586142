"""Multi-rank plumbing on CPU: world_size 2 over gloo.

Each rank scans its shard with an oracle-backed engine (the checker stands in
for the GPU kernels here, since there is no GPU), the product's ShardedSearch
all-gathers the per-shard top-k keys and merges them; the merged result must
equal the unsharded oracle search, ties included.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleEngine:
    """Per-shard search by the CPU oracle, emitting the same 64-bit keys as K2/K3."""

    def __init__(self, pq, codes, ids):
        self.pq, self.codes, self.ids = pq, codes, ids

    def search_keys(self, queries, params, keys, counts):
        import oracle
        oi, osc, oc, _, _ = oracle.search(self.pq, self.codes, queries.numpy(), int(params.k), tau=int(params.tau),
                                          ids=self.ids, threads=2)
        key = (osc.view(np.uint32).astype(np.uint64) << np.uint64(32)) | (oi.astype(np.uint64) & np.uint64(0xFFFFFFFF))
        key[oi < 0] = np.uint64(0xFFFFFFFFFFFFFFFF)
        keys.copy_(torch.from_numpy(key.view(np.int64)))
        counts.copy_(torch.from_numpy(oc.astype(np.int32)))

    def merge(self, keys_all, counts_all, parts, nq, k, ids, scores, counts):
        for q in range(nq):
            pool = []
            for p in range(parts):
                c = int(counts_all[p, q])
                pool.extend(int(x) & 0xFFFFFFFFFFFFFFFF for x in keys_all[p, q, :c].tolist())
            pool.sort()
            top = pool[:k]
            counts[q] = len(top)
            for r in range(k):
                if r < len(top):
                    ids[q, r] = top[r] & 0xFFFFFFFF
                    scores[q, r] = float(np.uint32(top[r] >> 32).view(np.float32))
                else:
                    ids[q, r] = -1
                    scores[q, r] = float("inf")


def _worker(rank, world, port, result_path, exchange="allgather"):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from conftest import load_pq
    from paper_1609_01882_b200.distributed import ShardedSearch, shard_range

    class P:  # SearchParams without importing the CUDA library
        k, tau = 30, 24

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_m8.npz"))
    pq = load_pq("pq_d128_m8.npz")
    codes = np.repeat(g["codes"][:3000], 2, axis=0)  # ties across the shard boundary
    b, e = shard_range(len(codes), world, rank)
    eng = OracleEngine(pq, codes[b:e], np.arange(b, e, dtype=np.int64))
    ids, scores, counts = ShardedSearch(eng, device="cpu", exchange=exchange).search_batch(
        torch.from_numpy(g["queries"]), P())
    if rank == 0:
        np.savez(result_path, ids=ids.numpy(), scores=scores.numpy(), counts=counts.numpy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("exchange", ["allgather", "alltoall"])
def test_sharded_search_equals_unsharded(tmp_path, pq8, g8, exchange):
    import oracle
    from paper_1609_01882_b200.distributed import shard_range
    assert [shard_range(10, 3, r) for r in range(3)] == [(0, 4), (4, 8), (8, 10)]
    out = str(tmp_path / "r0.npz")
    mp.spawn(_worker, args=(2, _free_port(), out, exchange), nprocs=2, join=True)
    r = np.load(out)
    codes = np.repeat(g8["codes"][:3000], 2, axis=0)
    oi, osc, oc, _, _ = oracle.search(pq8, codes, g8["queries"], 30, tau=24)
    assert np.array_equal(r["ids"], oi)
    assert np.array_equal(r["scores"].view(np.uint32), osc.view(np.uint32))
    assert np.array_equal(r["counts"], oc.astype(np.int32))


class OracleIVFEngine(OracleEngine):
    """IVF shard (every cell's list restricted to the rank's id range, coarse quantizer
    replicated) searched by the IVF oracle; same keys and merge as the flat engine."""

    def __init__(self, pq, coarse, lists, nprobe):
        self.pq, self.coarse, self.lists, self.nprobe = pq, coarse, lists, nprobe

    def search_keys(self, queries, params, keys, counts):
        import oracle
        oi, osc, oc, _, _, _ = oracle.ivf_search(self.pq, self.coarse, self.lists, queries.numpy(), int(params.k),
                                                 self.nprobe, tau=int(params.tau), threads=2)
        key = (osc.view(np.uint32).astype(np.uint64) << np.uint64(32)) | (oi.astype(np.uint64) & np.uint64(0xFFFFFFFF))
        key[oi < 0] = np.uint64(0xFFFFFFFFFFFFFFFF)
        keys.copy_(torch.from_numpy(key.view(np.int64)))
        counts.copy_(torch.from_numpy(oc.astype(np.int32)))


def _ivf_data():
    import oracle
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden_ivf.npz"))
    pq = oracle.PQ(8, 8, 128, g["codebooks"], g["perms"])
    centers = oracle.gen_centers(int(g["data_seed"]), 1000, 128)
    base = oracle.gen_points(int(g["data_seed"]), 2, 0, 20000, centers)
    base = np.concatenate([base, base[:500]])  # duplicates across the shard boundary: ties
    return g, pq, base


def _ivf_worker(rank, world, port, result_path):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1609_01882_b200.distributed import ShardedSearch, shard_range

    class P:
        k, tau = 40, 26

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g, pq, base = _ivf_data()
    b, e = shard_range(len(base), world, rank)
    lists, _ = oracle.ivf_build(pq, base[b:e], g["coarse"], ids=np.arange(b, e, dtype=np.int64))
    eng = OracleIVFEngine(pq, g["coarse"], lists, nprobe=8)
    ids, scores, counts = ShardedSearch(eng, device="cpu").search_batch(torch.from_numpy(g["queries"]), P())
    if rank == 0:
        np.savez(result_path, ids=ids.numpy(), scores=scores.numpy(), counts=counts.numpy())
    dist.destroy_process_group()


def test_sharded_ivf_equals_unsharded(tmp_path):
    """SURVEY.md sec. 8e for IVF on CPU: ids sharded within every list, same probes on
    every rank, keys all-gathered over gloo and merged == the unsharded IVF oracle."""
    import oracle
    out = str(tmp_path / "ivf0.npz")
    mp.spawn(_ivf_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    g, pq, base = _ivf_data()
    lists, _ = oracle.ivf_build(pq, base, g["coarse"])
    oi, osc, oc, _, _, _ = oracle.ivf_search(pq, g["coarse"], lists, g["queries"], 40, 8, tau=26)
    assert np.array_equal(r["ids"], oi)
    assert np.array_equal(r["scores"].view(np.uint32), osc.view(np.uint32))
    assert np.array_equal(r["counts"], oc.astype(np.int32))


def _ivf_bylist_worker(rank, world, port, result_path):
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_1609_01882_b200.distributed import ShardedSearch, assign_lists

    class P:
        k, tau = 40, 26

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g, pq, base = _ivf_data()
    cells = oracle.ivf_assign(base, g["coarse"], threads=2)
    owner = assign_lists(np.bincount(cells, minlength=len(g["coarse"])), world)
    rows = np.nonzero(owner[cells] == rank)[0]
    lists, _ = oracle.ivf_build(pq, base[rows], g["coarse"], ids=rows.astype(np.int64), assign=cells[rows])
    eng = OracleIVFEngine(pq, g["coarse"], lists, nprobe=8)
    ids, scores, counts = ShardedSearch(eng, device="cpu").search_batch(torch.from_numpy(g["queries"]), P())
    if rank == 0:
        np.savez(result_path, ids=ids.numpy(), scores=scores.numpy(), counts=counts.numpy(), owner=owner)
    dist.destroy_process_group()


def test_sharded_ivf_by_list_equals_unsharded(tmp_path):
    """SURVEY.md sec. 8e by-list sharding on CPU: each rank holds whole lists (assign_lists,
    balanced by size), the same probes on every rank, keys all-gathered over gloo and
    merged == the unsharded IVF oracle."""
    import oracle
    from paper_1609_01882_b200.distributed import assign_lists
    assert assign_lists([5, 1, 4, 4], 2).tolist() == [0, 0, 1, 1]  # LPT: 5 -> r0, 4 -> r1, 4 -> r1 (4 < 5), 1 -> r0
    out = str(tmp_path / "ivfl0.npz")
    mp.spawn(_ivf_bylist_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = np.load(out)
    assert set(np.unique(r["owner"])) == {0, 1}
    g, pq, base = _ivf_data()
    lists, _ = oracle.ivf_build(pq, base, g["coarse"])
    oi, osc, oc, _, _, _ = oracle.ivf_search(pq, g["coarse"], lists, g["queries"], 40, 8, tau=26)
    assert np.array_equal(r["ids"], oi)
    assert np.array_equal(r["scores"].view(np.uint32), osc.view(np.uint32))
    assert np.array_equal(r["counts"], oc.astype(np.int32))


def _gather_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist
    from paper_1609_01882_b200.distributed import gather_query_slices
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        q = torch.arange(7 * 3, dtype=torch.float32).reshape(7, 3)
        seen = []

        def compute(rows):  # order-sensitive: row sums as int64 probe-like keys, 2 columns
            seen.append(rows.shape[0])
            s = rows.sum(1).to(torch.int64)
            return torch.stack([s, s * 10], 1)

        out = gather_query_slices(compute, q)
        want = torch.stack([q.sum(1).to(torch.int64), q.sum(1).to(torch.int64) * 10], 1)
        if rank == 0:
            torch.save({"ok": bool(torch.equal(out, want)), "rows": seen}, result_path)
    finally:
        dist.destroy_process_group()


def test_gather_query_slices(tmp_path):
    """The query-split coarse quantization's gather: each rank computes its slice of
    the queries (shard_range), the all-gather returns every row in query order."""
    import torch
    import torch.multiprocessing as mp
    out = str(tmp_path / "gather.pt")
    mp.spawn(_gather_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    r = torch.load(out)
    assert r["ok"] and r["rows"] == [4]
