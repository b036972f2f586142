"""IVF + polysemous index (SPEC.md coarseindex, :350-417) over the C ABI.

Names follow the SPEC operations: ``assign`` / ``add`` (build, :370-375),
``probes`` (enumerate_cells, :376-381) and ``search`` (search_coarse,
:382-390, with nprobe and the pre-filter candidate cap).  The reference
ships no code for this module; parity is against the oracle restatement
pinned to golden vectors composed from the reference's primitives.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import IvfParamsC, PqDesc, SearchStatsC, lib
from .flat_index import Errc, PolyError, ProductQuantizer, SearchStats, Strategy, _check, _p


@dataclass
class CoarseParams:
    """SearchParams + CoarseConfig: k, tau, strategy, nprobe, cap (0 = none)."""
    strategy: Strategy = Strategy.dual
    k: int = 10
    tau: int = 0
    nprobe: int = 1
    cap: int = 0

    def c(self):
        return IvfParamsC(int(self.strategy), int(self.k), int(self.tau), int(self.nprobe), int(self.cap))


class IVFIndex:
    """Inverted file over residual polysemous codes on one B200."""

    def __init__(self, pq: ProductQuantizer, coarse, device: int = 0, _handle=None):
        self._pq = pq
        self.device = device
        self.coarse = np.ascontiguousarray(coarse, np.float32).reshape(-1, pq.dim)
        self.nlist = self.coarse.shape[0]
        if _handle is not None:
            self._h = _handle
            return
        d = PqDesc(pq.m, pq.dbits, pq.dim, _p(pq.codebooks), _p(pq.perms))
        h = C.c_void_p()
        _check(lib.poly_b200_ivf_create(C.byref(d), _p(self.coarse), self.nlist, device, C.byref(h)))
        self._h = h

    # ---- inverted-list file (layout in ivf_format.py)
    def save(self, path):
        _check(lib.poly_b200_ivf_save(self._h, str(path).encode()))

    @classmethod
    def load(cls, path, device: int = 0):
        from .ivf_format import read_header_tables
        h = C.c_void_p()
        _check(lib.poly_b200_ivf_load(str(path).encode(), device, C.byref(h)))
        m, dim, codebooks, perms, coarse = read_header_tables(path)
        return cls(ProductQuantizer(m, 8, dim, codebooks, perms), coarse, device, _handle=h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib.poly_b200_ivf_destroy(h)
            self._h = None

    def pq(self):
        return self._pq

    def size(self) -> int:
        return int(lib.poly_b200_ivf_size(self._h))

    def assign(self, x):
        x = np.ascontiguousarray(x, np.float32).reshape(-1, self._pq.dim)
        out = np.empty(x.shape[0], np.uint32)
        _check(lib.poly_b200_ivf_assign(self._h, _p(x), x.shape[0], _p(out)))
        return out

    def add(self, x, ids=None, cells=None):
        x = np.ascontiguousarray(x, np.float32)
        if x.ndim != 2 or x.shape[1] != self._pq.dim:
            raise PolyError(Errc.invalid_argument, "encode dimension mismatch")
        ids = None if ids is None else np.ascontiguousarray(ids, np.int64)
        cells = None if cells is None else np.ascontiguousarray(cells, np.uint32)
        _check(lib.poly_b200_ivf_add(self._h, _p(x), x.shape[0], _p(cells), _p(ids)))

    def add_device(self, d_x, d_cells, id0, stream=0):
        _check(lib.poly_b200_ivf_add_device(self._h, d_x.data_ptr(), d_cells.data_ptr(), d_x.shape[0], int(id0),
                                            C.c_void_p(stream)))

    def add_device_ids(self, d_x, d_cells, ids, stream=0):
        """add_device with explicit (host, int64) ids."""
        ids = np.ascontiguousarray(ids, np.int64)
        _check(lib.poly_b200_ivf_add_device_ids(self._h, d_x.data_ptr(), d_cells.data_ptr(), d_x.shape[0], _p(ids),
                                                C.c_void_p(stream)))

    def add_codes(self, cells, codes, ids=None):
        cells = np.ascontiguousarray(cells, np.uint32)
        codes = np.ascontiguousarray(codes, np.uint8)
        ids = None if ids is None else np.ascontiguousarray(ids, np.int64)
        _check(lib.poly_b200_ivf_add_codes(self._h, _p(cells), _p(codes), _p(ids), cells.shape[0]))

    def lists(self):
        """(off [nlist+1], codes [n, code_bytes], ids [n]) in list order."""
        n = self.size()
        off = np.empty(self.nlist + 1, np.uint64)
        codes = np.empty((n, self._pq.code_bytes()), np.uint8)
        ids = np.empty(n, np.int64)
        _check(lib.poly_b200_ivf_get_lists(self._h, _p(off), _p(codes), _p(ids)))
        return off, codes, ids

    def list_offsets(self):
        """CSR offsets [nlist+1] of the inverted lists (builds the lists if adds are pending)."""
        off = np.empty(self.nlist + 1, np.uint64)
        _check(lib.poly_b200_ivf_get_lists(self._h, _p(off), None, None))
        return off

    def probes(self, queries, nprobe):
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self._pq.dim)
        out = np.empty((q.shape[0], nprobe), np.uint32)
        _check(lib.poly_b200_ivf_probes(self._h, _p(q), q.shape[0], nprobe, _p(out)))
        return out

    def search(self, queries, params: CoarseParams, stats: SearchStats | None = None, out=None):
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self._pq.dim)
        nq, k = q.shape[0], int(params.k)
        if out is None:  # out: preallocated (e.g. pinned) ids [nq,k] int64, scores [nq,k] fp32, counts [nq] uint32
            out = (np.empty((nq, k), np.int64), np.empty((nq, k), np.float32), np.empty(nq, np.uint32))
        ids, scores, counts = out
        st = SearchStatsC()
        _check(lib.poly_b200_ivf_search(self._h, _p(q), nq, C.byref(params.c()), _p(ids), _p(scores), _p(counts),
                                        C.byref(st)))
        if stats is not None:
            stats.scanned += st.scanned
            stats.survivors += st.survivors
        return ids, scores, counts

    def search_device(self, d_queries, params: CoarseParams, d_ids, d_scores, d_counts=None, stream=0,
                      stats: SearchStats | None = None, d_survivors=None, d_survivor_hash=None):
        """Device buffers (torch CUDA tensors).  ``d_survivors`` / ``d_survivor_hash``:
        per-query survivor counts and sum of mix64(id) over the survivors (stats mode)."""
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        st = SearchStatsC()
        _check(lib.poly_b200_ivf_search_device_ex(self._h, ptr(d_queries), d_queries.shape[0], C.byref(params.c()),
                                                  ptr(d_ids), ptr(d_scores), ptr(d_counts), ptr(d_survivors),
                                                  ptr(d_survivor_hash), C.c_void_p(stream),
                                                  C.byref(st) if stats is not None else None))
        if stats is not None:
            stats.scanned += st.scanned
            stats.survivors += st.survivors

    def cells(self, cells):
        """CSR of the given cells' lists: (off [len+1] uint64, codes [off[-1], cb] uint8, ids int64)."""
        cells = np.ascontiguousarray(cells, np.uint32)
        off = np.empty(len(cells) + 1, np.uint64)
        _check(lib.poly_b200_ivf_get_cells(self._h, _p(cells), len(cells), _p(off), None, None))
        codes = np.empty((int(off[-1]), self._pq.code_bytes()), np.uint8)
        ids = np.empty(int(off[-1]), np.int64)
        _check(lib.poly_b200_ivf_get_cells(self._h, _p(cells), len(cells), _p(off), _p(codes), _p(ids)))
        return off, codes, ids

    def profile_enable(self, on: bool = True):
        _check(lib.poly_b200_ivf_profile_enable(self._h, int(on)))

    def profile_read(self):
        """(summed K6 list-scan milliseconds, K6 launches) since the last read."""
        ms, n = C.c_double(0), C.c_uint64(0)
        _check(lib.poly_b200_ivf_profile_read(self._h, C.byref(ms), C.byref(n)))
        return float(ms.value), int(n.value)

    def set_batch(self, queries_per_batch: int):
        """Queries per internal batch (default 2048); larger batches share list reads."""
        _check(lib.poly_b200_ivf_set_batch(self._h, int(queries_per_batch)))

    @property
    def batch(self) -> int:
        return int(lib.poly_b200_ivf_batch(self._h))

    def debug_set_list_capacity(self, cap: int):
        _check(lib.poly_b200_ivf_debug_set_list_capacity(self._h, int(cap)))

    def debug_rescued(self) -> int:
        n = C.c_uint32(0)
        _check(lib.poly_b200_ivf_debug_rescued(self._h, C.byref(n)))
        return int(n.value)

    def search_keys_device(self, d_queries, params: CoarseParams, d_keys, d_counts, stream=0,
                           stats: SearchStats | None = None, probes=None):
        """Multi-GPU: this shard's top-k as int64 keys (score bits << 32 | global id).
        probes: optional nq x min(nprobe, nlist) int64 probe keys (probe_keys_device),
        e.g. all-gathered from the ranks that each enumerated a query slice."""
        st = SearchStatsC()
        stp = C.byref(st) if stats is not None else None
        if probes is None:
            _check(lib.poly_b200_ivf_search_keys_device(self._h, d_queries.data_ptr(), d_queries.shape[0],
                                                        C.byref(params.c()), d_keys.data_ptr(), d_counts.data_ptr(),
                                                        C.c_void_p(stream), stp))
        else:
            _check(lib.poly_b200_ivf_search_keys_probes_device(
                self._h, d_queries.data_ptr(), d_queries.shape[0], C.byref(params.c()), probes.data_ptr(),
                d_keys.data_ptr(), d_counts.data_ptr(), C.c_void_p(stream), stp))
        if stats is not None:
            stats.scanned += st.scanned
            stats.survivors += st.survivors

    def search_keys_phase_device(self, d_queries, params: CoarseParams, probes, phase, d_thr, d_keys=None,
                                 d_counts=None, stream=0, stats: SearchStats | None = None):
        """By-list sharding's two-phase shard search (poly_b200_ivf_search_keys_phase_device):
        phase 1 writes the local round-1 bound to d_thr (nq uint64 as int64); after the
        caller's min-reduce, phase 2 reads it and writes this shard's top-k keys."""
        st = SearchStatsC()
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        _check(lib.poly_b200_ivf_search_keys_phase_device(
            self._h, d_queries.data_ptr(), d_queries.shape[0], C.byref(params.c()), probes.data_ptr(), int(phase),
            d_thr.data_ptr(), ptr(d_keys), ptr(d_counts), C.c_void_p(stream), C.byref(st) if stats is not None else None))
        if stats is not None:
            stats.scanned += st.scanned
            stats.survivors += st.survivors

    def probe_keys_device(self, d_queries, nprobe, d_out, stream=0):
        """enumerate_cells on the GPU: nq x min(nprobe, nlist) int64 keys (dist bits << 32 | cell)."""
        _check(lib.poly_b200_ivf_probe_keys_device(self._h, d_queries.data_ptr(), d_queries.shape[0], int(nprobe),
                                                   d_out.data_ptr(), C.c_void_p(stream)))

    def merge_keys_device(self, d_keys, d_counts, parts, nq, k, d_ids, d_scores, d_counts_out=None, stream=0):
        """Exact merge of parts x nq x k keys (all ranks' search_keys_device output)."""
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        _check(lib.poly_b200_ivf_merge_keys_device(self._h, ptr(d_keys), ptr(d_counts), parts, nq, k, ptr(d_ids),
                                                   ptr(d_scores), ptr(d_counts_out), C.c_void_p(stream)))

    def knn_graph_write_device(self, writer: "KnnGraphWriter", d_x, id0, params: CoarseParams, stream=0):
        """knn_graph rows of the stored vectors d_x (ids id0..) appended to a graph file."""
        _check(lib.poly_b200_ivf_knn_graph_write_device(self._h, writer._w, d_x.data_ptr(), d_x.shape[0], int(id0),
                                                        C.byref(params.c()), C.c_void_p(stream)))

    def knn_graph_device(self, d_x, id0, params: CoarseParams, d_ids, d_scores, d_counts=None, stream=0):
        """knn_graph: rows of d_x are the stored vectors id0.. ; self-match removed."""
        ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
        _check(lib.poly_b200_ivf_knn_graph_device(self._h, ptr(d_x), d_x.shape[0], int(id0), C.byref(params.c()),
                                                  ptr(d_ids), ptr(d_scores), ptr(d_counts), C.c_void_p(stream)))


def kmeans(x, k: int, iters: int = 25, seed: int = 1234567, device: int = 0):
    """train_coarse's k-means on the GPU (kmeans.cpp:14-137 restated,
    KmeansParams defaults).  Returns (centroids k x dim, assign n, iteration_mse, mse)."""
    x = np.ascontiguousarray(x, np.float32)
    n, dim = x.shape
    cent = np.empty((k, dim), np.float32)
    assign = np.empty(n, np.uint32)
    it = np.zeros(max(iters, 1), np.float64)
    mse = C.c_double(0)
    _check(lib.poly_b200_kmeans(_p(x), n, dim, k, iters, seed, device, _p(cent), _p(assign), _p(it), C.byref(mse)))
    return cent, assign, it[:iters] if n > k else it[:0], float(mse.value)


class KnnGraphWriter:
    """The k-NN graph output sink: a sectioned binary graph file plus an
    optional ivecs export (layout in knn_format.py).  Use as a context manager."""

    def __init__(self, path, k: int, ivecs_path=None):
        w = C.c_void_p()
        _check(lib.poly_b200_knn_writer_open(str(path).encode(), None if ivecs_path is None else str(ivecs_path).encode(),
                                             int(k), C.byref(w)))
        self._w = w
        self.records = 0

    def close(self) -> int:
        if self._w:
            n = C.c_uint64(0)
            w, self._w = self._w, None
            _check(lib.poly_b200_knn_writer_close(w, C.byref(n)))
            self.records = int(n.value)
        return self.records

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
