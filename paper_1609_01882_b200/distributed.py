"""Database sharding across ranks (one process per GPU) with an exact top-k merge.

The flat index partitions naturally: rank r holds the
contiguous id range ``shard_range(N, world, r)`` and scans it; the only exchange
is one all-gather per query batch of each rank's top-k as 64-bit keys
(fp32 score bits << 32 | id rank), merged by the K3 kernel.  Keys carry global
id ranks, so the merge is exact, ties included.

The engine is pluggable so that the rank plumbing (ranges, gather layout,
merge order) is testable on CPU with gloo: ``FlatIndexEngine`` is the GPU
engine (C ABI); tests plug an oracle-backed engine.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, world: int, rank: int):
    """Contiguous [begin, end) of rank's shard; ceil-sized shards, last one shorter."""
    per = (n_total + world - 1) // world
    begin = min(rank * per, n_total)
    return begin, min(begin + per, n_total)


def assign_lists(list_sizes, world: int):
    """By-list sharding of an IVF index ("sharding by list"): the owner
    rank of every cell, cells placed largest first on the least loaded rank (ties to the
    lower rank), so each rank holds about 1/world of the codes.  Deterministic, so every
    rank computes the same table from the same list sizes."""
    import heapq

    import numpy as np
    sizes = np.asarray(list_sizes, np.int64)
    owner = np.empty(len(sizes), np.int32)
    heap = [(0, r) for r in range(world)]
    for c in np.argsort(-sizes, kind="stable"):
        load, r = heapq.heappop(heap)
        owner[c] = r
        heapq.heappush(heap, (load + int(sizes[c]), r))
    return owner


def by_list_balance(list_sizes, probe_cells, owner, world: int):
    """Per-rank codes scanned for a query batch under by-list sharding (probe_cells: nq x
    nprobe cells): (max / mean) -- the imbalance factor of the scan -- and the per-rank
    totals."""
    import numpy as np
    sizes = np.asarray(list_sizes, np.int64)
    cells = np.asarray(probe_cells, np.int64).ravel()
    per = np.bincount(np.asarray(owner)[cells], weights=sizes[cells], minlength=world)
    return float(per.max() / max(per.mean(), 1e-30)), per


class FlatIndexEngine:
    """GPU engine over one rank's FlatIndex shard.  Every call is enqueued on torch's
    current stream, the stream the all-gathers and the caching allocator use too, so
    the engine's kernels, the collectives and buffer reuse are ordered without extra
    events."""

    def __init__(self, index):
        self.index = index

    @staticmethod
    def _sptr():
        return torch.cuda.current_stream().cuda_stream

    def search_keys(self, queries, params, keys, counts):
        self.index.search_keys_device(queries, params, keys, counts, None, stream=self._sptr())

    def merge(self, keys_all, counts_all, parts, nq, k, ids, scores, counts):
        self.index.merge_keys_device(keys_all, counts_all, parts, nq, k, ids, scores, counts, stream=self._sptr())


def gather_query_slices(compute, queries, group=None):
    """Split the rows of ``queries`` over the ranks (``shard_range``), run
    ``compute(rows) -> tensor [len(rows), ...]`` on this rank's slice and all-gather
    the slices back into one [nq, ...] tensor, in query order, on every rank.  Slices
    are padded to the ceil size for the equal-size all-gather."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    nq = queries.shape[0]
    if world == 1:
        return compute(queries)
    per = (nq + world - 1) // world
    b, e = shard_range(nq, world, rank)
    part = compute(queries[b:e]) if e > b else None
    shape = (per,) + tuple(part.shape[1:] if part is not None else compute(queries[:1]).shape[1:])
    buf = torch.zeros(shape, dtype=part.dtype if part is not None else torch.int64, device=queries.device)
    if part is not None:
        buf[:e - b] = part
    out = torch.empty((world * per,) + shape[1:], dtype=buf.dtype, device=queries.device)
    dist.all_gather_into_tensor(out, buf, group=group)
    return out[:nq]


class IVFIndexEngine(FlatIndexEngine):
    """GPU engine over one rank's IVF shard.  Two shardings, the same
    engine code: by id (every cell's list restricted to the rank's id range) or by list
    (the rank holds whole lists, ``assign_lists``; the other cells' lists are empty here,
    so the rank builds residual LUTs and scans only for the probes that hit its own
    lists).  All ranks see the same probes and the key merge is exact either way.  With
    ``split_coarse`` the coarse quantization (tensor-core dots + exact re-rank) is split
    by query: each rank enumerates the probes of its query slice and the probe keys are
    all-gathered, instead of every rank enumerating every query."""

    def __init__(self, index, stats=None, split_coarse=False, group=None, by_list=False):
        super().__init__(index)
        self.stats = stats
        self.split_coarse = split_coarse or by_list
        self.group = group
        self.by_list = by_list

    def probe_keys(self, queries, nprobe):
        npr = min(int(nprobe), self.index.nlist)

        def compute(rows):
            out = torch.empty((rows.shape[0], npr), dtype=torch.int64, device=rows.device)
            if rows.shape[0]:
                self.index.probe_keys_device(rows, npr, out, stream=self._sptr())
            return out

        return gather_query_slices(compute, queries, self.group)

    def search_keys(self, queries, params, keys, counts):
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        if int(getattr(params, "cap", 0)) and world > 1:
            # the cap cuts a query's probe list where the codes scanned reach it; each rank
            # only sees its own slice of every list, so the cut would differ per rank
            from .flat_index import Errc, PolyError
            raise PolyError(Errc.invalid_argument, "CoarseParams.cap > 0 is not supported with sharded lists")
        probes = self.probe_keys(queries, params.nprobe) if self.split_coarse else None
        if not self.by_list:
            self.index.search_keys_device(queries, params, keys, counts, stream=self._sptr(), stats=self.stats,
                                          probes=probes)
            return
        # by-list: round 1 on the owner of each query's first probe, the bounds min-reduced
        # over the ranks, round 2 everywhere under the global bound (one batch per call)
        B = self.index.batch
        for b in range(0, queries.shape[0], B):
            q, pr = queries[b:b + B], probes[b:b + B]
            thr = torch.empty(q.shape[0], dtype=torch.int64, device=queries.device)
            self.index.search_keys_phase_device(q, params, pr, 1, thr, stream=self._sptr())
            if world > 1:
                # keys are < 2^63; 'no bound' (all ones = -1 as int64) -> INT64_MAX for the MIN
                thr = torch.where(thr == -1, torch.full_like(thr, 2**63 - 1), thr)
                dist.all_reduce(thr, op=dist.ReduceOp.MIN, group=self.group)
                thr = torch.where(thr == 2**63 - 1, torch.full_like(thr, -1), thr)
            self.index.search_keys_phase_device(q, params, pr, 2, thr, keys[b:b + B], counts[b:b + B],
                                                stream=self._sptr(), stats=self.stats)


class ShardedSearch:
    """search_batch over all ranks' shards: local scan, exchange of the per-shard top-k
    keys, exact merge.  ``exchange="allgather"``: every rank gathers every shard's keys and
    merges every query.  ``exchange="alltoall"``: rank r receives every shard's keys for its
    query slice only (shard_range over the queries), merges that slice, and the merged
    slices are all-gathered -- W x less key traffic and merge work per rank."""

    def __init__(self, engine, device="cuda", group=None, exchange="allgather"):
        self.engine = engine
        self.device = device
        self.group = group
        self.exchange = exchange
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def search_batch(self, queries, params, out=None):
        nq, k = queries.shape[0], int(params.k)
        dev = self.device
        if out is None:
            out = (torch.empty((nq, k), dtype=torch.int64, device=dev),
                   torch.empty((nq, k), dtype=torch.float32, device=dev),
                   torch.empty(nq, dtype=torch.int32, device=dev))
        keys = torch.empty((nq, k), dtype=torch.int64, device=dev)
        cnt = torch.empty(nq, dtype=torch.int32, device=dev)
        self.engine.search_keys(queries, params, keys, cnt)
        if self.world > 1 and self.exchange == "alltoall":
            return self._alltoall(keys, cnt, nq, k, out)
        if self.world == 1:
            keys_all, cnt_all = keys.unsqueeze(0), cnt.unsqueeze(0)
        else:
            # gathered along dim 0 (rank-major): parts x nq x k, the merge kernel's layout
            keys_all = torch.empty((self.world * nq, k), dtype=torch.int64, device=dev)
            cnt_all = torch.empty(self.world * nq, dtype=torch.int32, device=dev)
            dist.all_gather_into_tensor(keys_all, keys, group=self.group)
            dist.all_gather_into_tensor(cnt_all, cnt, group=self.group)
            keys_all = keys_all.view(self.world, nq, k)
            cnt_all = cnt_all.view(self.world, nq)
        self.engine.merge(keys_all, cnt_all, self.world, nq, k, *out)
        return out

    def _alltoall(self, keys, cnt, nq, k, out):
        W, dev = self.world, self.device
        rank = dist.get_rank(self.group)
        per = (nq + W - 1) // W
        # send block r = the rows of query slice r, padded to `per` rows (padding: count 0)
        send_k = torch.full((W * per, k), -1, dtype=torch.int64, device=dev)
        send_c = torch.zeros(W * per, dtype=torch.int32, device=dev)
        for r in range(W):
            b, e = shard_range(nq, W, r)
            send_k[r * per:r * per + (e - b)] = keys[b:e]
            send_c[r * per:r * per + (e - b)] = cnt[b:e]
        recv_k = torch.empty_like(send_k)
        recv_c = torch.empty_like(send_c)
        dist.all_to_all_single(recv_k, send_k, group=self.group)
        dist.all_to_all_single(recv_c, send_c, group=self.group)
        # recv block s = shard s's keys for this rank's slice: parts x per x k
        ids_s = torch.empty((per, k), dtype=torch.int64, device=dev)
        sc_s = torch.empty((per, k), dtype=torch.float32, device=dev)
        cnt_s = torch.empty(per, dtype=torch.int32, device=dev)
        self.engine.merge(recv_k.view(W, per, k), recv_c.view(W, per), W, per, k, ids_s, sc_s, cnt_s)
        ga = [torch.empty((W * per, k), dtype=torch.int64, device=dev),
              torch.empty((W * per, k), dtype=torch.float32, device=dev),
              torch.empty(W * per, dtype=torch.int32, device=dev)]
        for g, x in zip(ga, (ids_s, sc_s, cnt_s)):
            dist.all_gather_into_tensor(g, x, group=self.group)
        for r in range(W):
            b, e = shard_range(nq, W, r)
            for o, g in zip(out, ga):
                o[b:e] = g[r * per:r * per + (e - b)]
        del rank
        return out
