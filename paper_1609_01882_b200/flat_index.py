"""Python mirror of the reference's flat-index interface over the C ABI.

Mirrors /root/reference/proj/include/poly/flat_index.hpp:39-144 (Neighbor,
Strategy, SearchParams, SearchStats, FlatIndex) and pq.hpp:49-89
(ProductQuantizer fields) -- same names, same argument meaning, and the
reference's error classes (common.hpp:13-32) raised as ``PolyError``.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import PqDesc, SearchParamsC, SearchStatsC, lib


class Errc(enum.IntEnum):
    """poly::errc (common.hpp:13-22)."""
    ok = 0
    invalid_argument = 1
    io = 2
    format = 3
    state = 4
    corrupt = 5
    version = 6
    internal = 7


class PolyError(RuntimeError):
    """poly::error (common.hpp:25-32): message + error class."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = Errc(code)


def _check(rc: int):
    if rc != 0:
        raise PolyError(rc, lib.poly_b200_last_error().decode())


class Strategy(enum.IntEnum):
    """poly::Strategy (flat_index.hpp:44)."""
    adc = 0
    binary = 1
    disidx = 2
    dual = 3


def strategy_from_string(name: str) -> Strategy:
    try:
        return Strategy[name]
    except KeyError:
        raise PolyError(Errc.invalid_argument, f"unknown strategy '{name}'") from None


def to_string(s: Strategy) -> str:
    return Strategy(s).name


@dataclass
class SearchParams:
    """poly::SearchParams (flat_index.hpp:48-52)."""
    strategy: Strategy = Strategy.adc
    k: int = 10
    tau: int = 0

    def c(self):
        return SearchParamsC(int(self.strategy), int(self.k), int(self.tau))


@dataclass
class SearchStats:
    """poly::SearchStats (flat_index.hpp:54-57)."""
    scanned: int = 0
    survivors: int = 0


@dataclass
class Neighbor:
    """poly::Neighbor (flat_index.hpp:39-42)."""
    id: int
    score: float


class ProductQuantizer:
    """The fields of poly::ProductQuantizer (pq.hpp:49-89) the search path needs."""

    def __init__(self, m: int, dbits: int, dim: int, codebooks, perms):
        self.m, self.dbits, self.dim = int(m), int(dbits), int(dim)
        ks = 1 << self.dbits
        self.codebooks = np.ascontiguousarray(codebooks, dtype=np.float32).reshape(self.m, ks, self.dim // self.m)
        self.perms = np.ascontiguousarray(perms, dtype=np.uint16).reshape(self.m, ks)

    def ksub(self):
        return 1 << self.dbits

    def dsub(self):
        return self.dim // self.m

    def code_bits(self):
        return self.m * self.dbits

    def code_bytes(self):
        return (self.code_bits() + 7) // 8

    @classmethod
    def load(cls, path):
        z = np.load(path)
        return cls(int(z["m"]), int(z["dbits"]), int(z["dim"]), z["codebooks"], z["perms"])


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class FlatIndex:
    """poly::FlatIndex (flat_index.hpp:99-144) on one B200.

    ``search`` / ``search_batch`` run the fused GPU scan (csrc/kernels_scan.cu);
    results follow SPEC.md:303-317 exactly (two-pass dual semantics, top-k by
    (score, id) ascending, survivors-only on shortage).
    """

    def __init__(self, pq: ProductQuantizer, device: int = 0, _handle=None):
        self._pq = pq
        self.device = device
        self.default_tau = None  # flat_index.hpp:113 (set by calibrate, persisted)
        if _handle is not None:
            self._h = _handle
            return
        d = PqDesc(pq.m, pq.dbits, pq.dim, _p(pq.codebooks), _p(pq.perms))
        h = C.c_void_p()
        _check(lib.poly_b200_create(C.byref(d), device, C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.poly_b200_destroy(h)
            self._h = None

    # ---- accessors (flat_index.hpp:104-111)
    def pq(self):
        return self._pq

    def size(self) -> int:
        return int(lib.poly_b200_size(self._h))

    def __len__(self):
        return self.size()

    def code_bytes(self) -> int:
        return int(lib.poly_b200_code_bytes(self._h))

    def code_bits(self) -> int:
        return self._pq.code_bits()

    def codes(self):
        out = np.empty((self.size(), self.code_bytes()), np.uint8)
        _check(lib.poly_b200_get_codes(self._h, _p(out), None))
        return out

    def ids(self):
        out = np.empty(self.size(), np.int64)
        _check(lib.poly_b200_get_codes(self._h, None, _p(out)))
        return out

    # ---- add path (flat_index.hpp:115-119)
    def add(self, x, ids=None):
        x = np.ascontiguousarray(x, np.float32)
        if x.ndim != 2 or x.shape[1] != self._pq.dim:
            raise PolyError(Errc.invalid_argument, "encode dimension mismatch")
        ids = None if ids is None else np.ascontiguousarray(ids, np.int64)
        _check(lib.poly_b200_add(self._h, _p(x), x.shape[0], _p(ids)))

    def add_codes(self, codes, ids=None):
        codes = np.ascontiguousarray(codes, np.uint8)
        n = codes.shape[0] if codes.ndim == 2 else codes.size // self._pq.code_bytes()
        ids = None if ids is None else np.ascontiguousarray(ids, np.int64)
        _check(lib.poly_b200_add_codes(self._h, _p(codes), _p(ids), n))

    def add_synthetic(self, seed, centers, row0, n, stream_id=2, normalize=False):
        centers = np.ascontiguousarray(centers, np.float32)
        _check(lib.poly_b200_add_synthetic(self._h, seed, _p(centers), centers.shape[0], stream_id, row0, n,
                                           int(normalize)))

    # ---- search (flat_index.hpp:121-126)
    def search_batch(self, queries, params: SearchParams, stats: SearchStats | None = None, out=None):
        """Returns (ids [nq,k] int64, scores [nq,k] fp32, counts [nq] uint32)."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self._pq.dim)
        nq, k = q.shape[0], int(params.k)
        if out is None:  # out: preallocated (e.g. pinned) ids [nq,k] int64, scores [nq,k] fp32, counts [nq] uint32
            out = (np.empty((nq, k), np.int64), np.empty((nq, k), np.float32), np.empty(nq, np.uint32))
        ids, scores, counts = out
        st = SearchStatsC()
        _check(lib.poly_b200_search_batch(self._h, _p(q), nq, C.byref(params.c()), _p(ids), _p(scores), _p(counts),
                                          C.byref(st)))
        if stats is not None:
            stats.scanned += st.scanned
            stats.survivors += st.survivors
        return ids, scores, counts

    def search(self, query, params: SearchParams, stats: SearchStats | None = None):
        ids, scores, counts = self.search_batch(np.asarray(query, np.float32).reshape(1, -1), params, stats)
        return [Neighbor(int(ids[0, i]), float(scores[0, i])) for i in range(int(counts[0]))]

    def search_batch_device(self, d_queries, params: SearchParams, d_ids, d_scores, d_counts=None, d_survivors=None,
                            stream=0, stats: SearchStats | None = None, d_survivor_hash=None):
        """Device-resident variant: arguments are torch CUDA tensors (or raw pointers).
        ``d_survivors`` (per-query counts) / ``d_survivor_hash`` (per-query sum of
        mix64(id) over the filter survivors) select the per-query-stats scan variant;
        ``stats`` (totals) synchronises the stream."""
        ptr = lambda t: None if t is None else (t if isinstance(t, int) else t.data_ptr())  # noqa: E731
        nq = d_queries.shape[0]
        st = SearchStatsC()
        _check(lib.poly_b200_search_batch_device_ex(self._h, ptr(d_queries), nq, C.byref(params.c()), ptr(d_ids),
                                                    ptr(d_scores), ptr(d_counts), ptr(d_survivors),
                                                    ptr(d_survivor_hash), C.c_void_p(stream),
                                                    C.byref(st) if stats is not None else None))
        if stats is not None:
            stats.scanned += st.scanned
            stats.survivors += st.survivors

    def search_keys_device(self, d_queries, params: SearchParams, d_keys, d_counts, d_survivors=None, stream=0):
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        _check(lib.poly_b200_search_keys_device(self._h, ptr(d_queries), d_queries.shape[0], C.byref(params.c()),
                                                ptr(d_keys), ptr(d_counts), ptr(d_survivors), C.c_void_p(stream)))

    def merge_keys_device(self, d_keys, d_counts, parts, nq, k, d_ids, d_scores, d_counts_out=None, stream=0):
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        _check(lib.poly_b200_merge_keys_device(self._h, ptr(d_keys), ptr(d_counts), parts, nq, k, ptr(d_ids),
                                               ptr(d_scores), ptr(d_counts_out), C.c_void_p(stream)))

    # ---- test hooks: candidate-list overflow and its exact rescue (kernels_rescue.cu)
    def debug_set_list_capacity(self, cap: int):
        _check(lib.poly_b200_debug_set_list_capacity(self._h, int(cap)))

    def debug_rescued(self) -> int:
        n = C.c_uint32(0)
        _check(lib.poly_b200_debug_rescued(self._h, C.byref(n)))
        return int(n.value)

    # ---- K2 timing hook (bench.py)
    def profile_enable(self, on: bool = True):
        _check(lib.poly_b200_profile_enable(self._h, int(on)))

    def profile_read(self):
        """(summed K2 scan milliseconds, K2 launches) since the last read."""
        ms, n = C.c_double(0), C.c_uint64(0)
        _check(lib.poly_b200_profile_read(self._h, C.byref(ms), C.byref(n)))
        return float(ms.value), int(n.value)

    # ---- calibration / relabel (flat_index.hpp:128-136)
    def calibrate_threshold(self, train_queries, target_filter_rate: float):
        """Returns (tau, warning)."""
        q = np.ascontiguousarray(train_queries, np.float32).reshape(-1, self._pq.dim)
        tau, warn = C.c_uint32(0), C.c_int(0)
        _check(lib.poly_b200_calibrate_threshold(self._h, _p(q), q.shape[0], float(target_filter_rate),
                                                 C.byref(tau), C.byref(warn)))
        self.default_tau = int(tau.value)
        return int(tau.value), bool(warn.value)

    def with_assignments(self, perms):
        perms = np.ascontiguousarray(perms, np.uint16).reshape(self._pq.m, -1)
        h = C.c_void_p()
        _check(lib.poly_b200_with_assignments(self._h, _p(perms), C.byref(h)))
        pq = ProductQuantizer(self._pq.m, self._pq.dbits, self._pq.dim, self._pq.codebooks, perms)
        return FlatIndex(pq, self.device, _handle=h)


class ShardedFlatIndex:
    """One poly::FlatIndex over several GPUs of this process.

    ``devices`` lists one CUDA ordinal per shard (an ordinal may repeat).  Each
    add / add_codes call splits its rows into len(devices) contiguous parts, one
    per shard, ids kept global; search_batch runs every shard concurrently and
    merges the per-shard top-k lists on devices[0] (peer copies + an n-way
    (score, id) merge kernel): the results equal FlatIndex over the union.
    """

    def __init__(self, pq: ProductQuantizer, devices):
        self._pq = pq
        self.devices = [int(d) for d in devices]
        d = PqDesc(pq.m, pq.dbits, pq.dim, _p(pq.codebooks), _p(pq.perms))
        dev = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        _check(lib.poly_b200_sharded_create(C.byref(d), dev, len(self.devices), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.poly_b200_sharded_destroy(h)
            self._h = None

    def pq(self):
        return self._pq

    def size(self) -> int:
        return int(lib.poly_b200_sharded_size(self._h))

    def __len__(self):
        return self.size()

    def shard_sizes(self):
        out = []
        for g in range(int(lib.poly_b200_sharded_count(self._h))):
            n = C.c_uint64(0)
            _check(lib.poly_b200_sharded_shard_size(self._h, g, C.byref(n)))
            out.append(int(n.value))
        return out

    def add(self, x, ids=None):
        x = np.ascontiguousarray(x, np.float32)
        if x.ndim != 2 or x.shape[1] != self._pq.dim:
            raise PolyError(Errc.invalid_argument, "encode dimension mismatch")
        ids = None if ids is None else np.ascontiguousarray(ids, np.int64)
        _check(lib.poly_b200_sharded_add(self._h, _p(x), x.shape[0], _p(ids)))

    def add_codes(self, codes, ids=None):
        codes = np.ascontiguousarray(codes, np.uint8)
        n = codes.shape[0] if codes.ndim == 2 else codes.size // self._pq.code_bytes()
        ids = None if ids is None else np.ascontiguousarray(ids, np.int64)
        _check(lib.poly_b200_sharded_add_codes(self._h, _p(codes), _p(ids), n))

    def search_batch(self, queries, params: SearchParams, stats: SearchStats | None = None):
        """Returns (ids [nq,k] int64, scores [nq,k] fp32, counts [nq] uint32)."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self._pq.dim)
        nq, k = q.shape[0], int(params.k)
        ids, scores, counts = np.empty((nq, k), np.int64), np.empty((nq, k), np.float32), np.empty(nq, np.uint32)
        st = SearchStatsC()
        _check(lib.poly_b200_sharded_search_batch(self._h, _p(q), nq, C.byref(params.c()), _p(ids), _p(scores),
                                                  _p(counts), C.byref(st)))
        if stats is not None:
            stats.scanned += st.scanned
            stats.survivors += st.survivors
        return ids, scores, counts

    def search(self, query, params: SearchParams, stats: SearchStats | None = None):
        ids, scores, counts = self.search_batch(np.asarray(query, np.float32).reshape(1, -1), params, stats)
        return [Neighbor(int(ids[0, i]), float(scores[0, i])) for i in range(int(counts[0]))]


def debug_lut(index: FlatIndex, queries):
    """K1 only: (stored-field LUTs [nq,m,256], query codes [nq,code_bytes]) from the GPU."""
    q = np.ascontiguousarray(queries, np.float32).reshape(-1, index.pq().dim)
    lutp = np.empty((q.shape[0], index.pq().m, 256), np.float32)
    qc = np.empty((q.shape[0], index.code_bytes()), np.uint8)
    _check(lib.poly_b200_debug_lut(index._h, _p(q), q.shape[0], _p(lutp), _p(qc)))
    return lutp, qc


def launch_count() -> int:
    return int(lib.poly_b200_launch_count())


def gen_points_device(centers, seed, stream_id, row0, n, d_out, device=0, normalize=False, stream=0):
    centers = np.ascontiguousarray(centers, np.float32)
    _check(lib.poly_b200_gen_points_device(device, seed, _p(centers), centers.shape[0], centers.shape[1], stream_id,
                                           row0, n, int(normalize), d_out.data_ptr(), C.c_void_p(stream)))


__all__ = ["Errc", "PolyError", "Strategy", "SearchParams", "SearchStats", "Neighbor", "ProductQuantizer",
           "FlatIndex", "strategy_from_string", "to_string", "launch_count", "gen_points_device", "debug_lut", "_lib"]
