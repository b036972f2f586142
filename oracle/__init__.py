"""ctypes bindings for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Who may import this package: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``, only as the
checker or the timed CPU baseline.  The product package
``paper_1609_01882_b200`` never imports it.

Two libraries:

* ``oracle/build/libpolyoracle.so`` -- our C restatement (``polyoracle.c``),
  each function citing the reference file:line it restates.
* ``oracle/_ref/libpolyref.so`` -- the reference's own C++ sources compiled in
  place by ``oracle/Makefile`` plus ``ref_driver.cpp`` (C ABI glue).  Used to
  generate the golden fixtures that pin the restatement, and as the
  ``--impl reference`` CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libpolyoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpolyref.so")

STRATEGIES = {"adc": 0, "binary": 1, "disidx": 2, "dual": 3}

_P = C.c_void_p
_u32, _u64, _i32, _f64 = C.c_uint32, C.c_uint64, C.c_int, C.c_double


def build() -> None:
    """Compile the restatement (and the reference when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.po_gen_centers.argtypes = [_u64, _u32, _u32, _P]
        L.po_gen_points.argtypes = [_u64, _u32, _u64, _u64, _P, _u32, _u32, _i32, _P]
        L.po_hash64.argtypes = [_u64]
        L.po_hash64.restype = _u64
        L.po_sq_l2.argtypes = [_P, _P, C.c_size_t]
        L.po_sq_l2.restype = C.c_float
        L.po_hamming_bytes.argtypes = [_P, _P, C.c_size_t]
        L.po_hamming_bytes.restype = _u32
        L.po_disidx.argtypes = [_P, _P, _u32, _u32]
        L.po_disidx.restype = _u32
        L.po_topk_select.argtypes = [_P, _P, _u64, _u32, _P, _P]
        L.po_topk_select.restype = _u32
        L.po_search_batch.argtypes = [_u32, _u32, _u32, _P, _P, _P, _P, _P, _u64, _P, _u64, _i32, _u32, _u32,
                                      C.c_uint, _P, _P, _P, _P, _P]
        L.po_search_batch.restype = _i32
        L.po_encode_batch.argtypes = [_u32, _u32, _u32, _P, _P, _P, _u64, _P, C.c_uint]
        L.po_lut_batch.argtypes = [_u32, _u32, _u32, _P, _P, _P, _P, _u64, _P, _P, _P]
        L.po_hamming_histogram.argtypes = [_u32, _u32, _u32, _P, _P, _P, _u64, _P, _u64, C.c_uint, _P]
        L.po_calibrate_from_histogram.argtypes = [_P, _u64, _u32, _u64, _f64, C.POINTER(_i32)]
        L.po_calibrate_from_histogram.restype = _u32
        L.po_relabel_codes.argtypes = [_u32, _u32, _P, _P, _P, _u64]
        L.po_ivf_assign.argtypes = [_P, _u64, _u32, _P, _u32, C.c_uint, _P]
        L.po_ivf_search.argtypes = [_u32, _u32, _u32, _P, _P, _P, _P, _u32, _P, _P, _P, _P, _u64, _u32, _u64, _i32,
                                    _u32, _u32, C.c_uint, _P, _P, _P, _P, _P, _P, _P]
        L.po_ivf_search.restype = _i32
        L.po_ivf_encode_residuals.argtypes = [_u32, _u32, _u32, _P, _P, _P, _u64, _P, _P, _P]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference; run make -C oracle)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_train_pq.argtypes = [_P, _u64, _u64, _u32, _u32, _u32, _u64, C.c_uint, _P]
        L.ref_optimize_pq.argtypes = [_u32, _u32, _u64, _P, _i32, _f64, _u64, _u64, C.c_uint, _P]
        L.ref_encode.argtypes = [_u32, _u32, _u64, _P, _P, _P, _u64, _P]
        L.ref_encode_batch.argtypes = [_u32, _u32, _u64, _P, _P, _P, _u64, _P, C.c_uint]
        L.ref_compute_lut.argtypes = [_u32, _u32, _u64, _P, _P, _P, _u64, _P, _P]
        L.ref_adc_matrix.argtypes = [_u32, _u32, _u64, _P, _P, _P, _u64, _P, _u64, _P]
        L.ref_hamming_matrix.argtypes = [_P, _u64, _P, _u64, _u64, _P]
        L.ref_hamming_matrix.restype = None
        L.ref_search_batch.argtypes = [_u32, _u32, _u64, _P, _P, _P, _P, _u64, _P, _u64, _i32, _u32, _u32, C.c_uint,
                                       _P, _P, _P, _P]
        L.ref_buggy_topk.argtypes = [_P, _P, _u64, _u32, _P, _P]
        L.ref_kmeans.argtypes = [_P, _u64, _u64, _u32, _u32, _u64, _P]
        L.ref_assign_nearest.argtypes = [_P, _u64, _P, _u64, _u64, _P]
        L.ref_ivf_search.argtypes = [_u32, _u32, _u64, _P, _P, _P, _u32, _P, _P, _P, _P, _u64, _u32, _u64, _i32, _u32,
                                     _u32, C.c_uint, _P, _P, _P, _P]
        L.ref_buggy_topk.restype = _u32
        _ref = L
    return _ref


def _check_ref(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {ref().ref_last_error().decode()}")


# --------------------------------------------------------------------------- PQ container
class PQ:
    """Codebooks + assignments, mirroring poly::ProductQuantizer (pq.hpp:49-89)."""

    def __init__(self, m, dbits, dim, codebooks, perms):
        self.m, self.dbits, self.dim = int(m), int(dbits), int(dim)
        ks = 1 << self.dbits
        self.codebooks = np.ascontiguousarray(codebooks, dtype=np.float32).reshape(self.m, ks, self.dim // self.m)
        self.perms = np.ascontiguousarray(perms, dtype=np.uint16).reshape(self.m, ks)
        inv = np.empty_like(self.perms)
        for sq in range(self.m):
            inv[sq, self.perms[sq]] = np.arange(ks, dtype=np.uint16)
        self.inv_perms = inv

    @property
    def code_bits(self):
        return self.m * self.dbits

    @property
    def code_bytes(self):
        return (self.code_bits + 7) // 8

    def args(self):
        return (self.m, self.dbits, self.dim, _ptr(self.codebooks), _ptr(self.perms))


# --------------------------------------------------------------------------- generator
def gen_centers(seed, ncent, dim):
    out = np.empty((ncent, dim), np.float32)
    lib().po_gen_centers(seed, ncent, dim, _ptr(out))
    return out


def gen_points(seed, stream, row0, n, centers, normalize=False):
    centers = np.ascontiguousarray(centers, np.float32)
    ncent, dim = centers.shape
    out = np.empty((n, dim), np.float32)
    lib().po_gen_points(seed, stream, row0, n, _ptr(centers), ncent, dim, int(normalize), _ptr(out))
    return out


# --------------------------------------------------------------------------- restatement
def encode(pq: PQ, x, threads=8):
    x = np.ascontiguousarray(x, np.float32)
    codes = np.empty((x.shape[0], pq.code_bytes), np.uint8)
    lib().po_encode_batch(*pq.args(), _ptr(x), x.shape[0], _ptr(codes), threads)
    return codes


def lut_batch(pq: PQ, q):
    q = np.ascontiguousarray(q, np.float32)
    nq = q.shape[0]
    ks = 1 << pq.dbits
    lut = np.empty((nq, pq.m, ks), np.float32)
    lutp = np.empty((nq, pq.m, ks), np.float32)
    qc = np.empty((nq, pq.code_bytes), np.uint8)
    lib().po_lut_batch(*pq.args(), _ptr(pq.inv_perms), _ptr(q), nq, _ptr(lut), _ptr(lutp), _ptr(qc))
    return lut, lutp, qc


def search(pq: PQ, codes, queries, k, tau=None, strategy="dual", ids=None, threads=8):
    """Two-pass dual search.  Returns ids, scores, counts, survivors, survivor_hash."""
    codes = np.ascontiguousarray(codes, np.uint8)
    queries = np.ascontiguousarray(queries, np.float32)
    n, nq = codes.shape[0], queries.shape[0]
    if ids is None:
        ids = np.arange(n, dtype=np.int64)
    ids = np.ascontiguousarray(ids, np.int64)
    tau = pq.code_bits if tau is None else tau
    oi = np.empty((nq, k), np.int64)
    osc = np.empty((nq, k), np.float32)
    oc = np.empty(nq, np.uint32)
    sv = np.empty(nq, np.uint64)
    sh = np.empty(nq, np.uint64)
    rc = lib().po_search_batch(*pq.args(), _ptr(pq.inv_perms), _ptr(codes), _ptr(ids), n, _ptr(queries), nq,
                               STRATEGIES[strategy], k, tau, threads, _ptr(oi), _ptr(osc), _ptr(oc), _ptr(sv), _ptr(sh))
    if rc != 0:
        raise ValueError(f"oracle search rejected arguments (rc={rc})")
    return oi, osc, oc, sv, sh


def topk_select(scores, ids, k):
    scores = np.ascontiguousarray(scores, np.float32)
    ids = np.ascontiguousarray(ids, np.int64)
    oi = np.empty(max(k, 1), np.int64)
    osc = np.empty(max(k, 1), np.float32)
    n = lib().po_topk_select(_ptr(scores), _ptr(ids), scores.shape[0], k, _ptr(oi), _ptr(osc))
    return oi[:n], osc[:n]


def hamming_histogram(pq: PQ, codes, queries, threads=8):
    codes = np.ascontiguousarray(codes, np.uint8)
    queries = np.ascontiguousarray(queries, np.float32)
    hist = np.empty((queries.shape[0], pq.code_bits + 1), np.uint64)
    lib().po_hamming_histogram(*pq.args(), _ptr(codes), codes.shape[0], _ptr(queries), queries.shape[0], threads,
                               _ptr(hist))
    return hist


def calibrate_threshold(pq: PQ, codes, train_queries, rate, threads=8):
    hist = hamming_histogram(pq, codes, train_queries, threads)
    w = _i32(0)
    tau = lib().po_calibrate_from_histogram(_ptr(hist), hist.shape[0], pq.code_bits, codes.shape[0], rate,
                                            C.byref(w))
    return int(tau), bool(w.value)


def relabel_codes(pq_old: PQ, new_perms, codes):
    out = np.array(codes, np.uint8, copy=True)
    new_perms = np.ascontiguousarray(new_perms, np.uint16)
    lib().po_relabel_codes(pq_old.m, pq_old.dbits, _ptr(pq_old.inv_perms), _ptr(new_perms), _ptr(out), out.shape[0])
    return out


def hamming(a, b):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    return int(lib().po_hamming_bytes(_ptr(a), _ptr(b), a.shape[-1]))


# --------------------------------------------------------------------------- reference
def ref_train_pq(train, m, dbits=8, iters=25, seed=1234567, threads=0):
    train = np.ascontiguousarray(train, np.float32)
    n, dim = train.shape
    cb = np.empty((m, 1 << dbits, dim // m), np.float32)
    _check_ref(ref().ref_train_pq(_ptr(train), n, dim, m, dbits, iters, seed, threads, _ptr(cb)))
    return cb


def ref_optimize_pq(codebooks, dim, dbits=8, loss=0, alpha=0.5, n_iter=500000, seed=1234567, threads=0):
    codebooks = np.ascontiguousarray(codebooks, np.float32)
    m = codebooks.shape[0]
    perms = np.empty((m, 1 << dbits), np.uint16)
    _check_ref(ref().ref_optimize_pq(m, dbits, dim, _ptr(codebooks), loss, alpha, n_iter, seed, threads, _ptr(perms)))
    return perms


def ref_encode(pq: PQ, x):
    x = np.ascontiguousarray(x, np.float32)
    codes = np.empty((x.shape[0], pq.code_bytes), np.uint8)
    _check_ref(ref().ref_encode(*pq.args(), _ptr(x), x.shape[0], _ptr(codes)))
    return codes


def ref_encode_batch(pq: PQ, x, threads=0):
    x = np.ascontiguousarray(x, np.float32)
    codes = np.empty((x.shape[0], pq.code_bytes), np.uint8)
    _check_ref(ref().ref_encode_batch(*pq.args(), _ptr(x), x.shape[0], _ptr(codes), threads))
    return codes


def ref_compute_lut(pq: PQ, q):
    q = np.ascontiguousarray(q, np.float32)
    nq = q.shape[0]
    lut = np.empty((nq, pq.m, 1 << pq.dbits), np.float32)
    lutp = np.empty_like(lut)
    _check_ref(ref().ref_compute_lut(*pq.args(), _ptr(q), nq, _ptr(lut), _ptr(lutp)))
    return lut, lutp


def ref_adc_matrix(pq: PQ, q, codes):
    q = np.ascontiguousarray(q, np.float32)
    codes = np.ascontiguousarray(codes, np.uint8)
    out = np.empty((q.shape[0], codes.shape[0]), np.float32)
    _check_ref(ref().ref_adc_matrix(*pq.args(), _ptr(q), q.shape[0], _ptr(codes), codes.shape[0], _ptr(out)))
    return out


def ref_hamming_matrix(a, b):
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    out = np.empty((a.shape[0], b.shape[0]), np.uint32)
    ref().ref_hamming_matrix(_ptr(a), a.shape[0], _ptr(b), b.shape[0], a.shape[1], _ptr(out))
    return out


def ref_search(pq: PQ, codes, queries, k, tau=None, strategy="dual", ids=None, threads=0):
    codes = np.ascontiguousarray(codes, np.uint8)
    queries = np.ascontiguousarray(queries, np.float32)
    n, nq = codes.shape[0], queries.shape[0]
    ids = np.arange(n, dtype=np.int64) if ids is None else np.ascontiguousarray(ids, np.int64)
    tau = pq.code_bits if tau is None else tau
    oi = np.empty((nq, k), np.int64)
    osc = np.empty((nq, k), np.float32)
    oc = np.empty(nq, np.uint32)
    sv = np.empty(nq, np.uint64)
    _check_ref(ref().ref_search_batch(*pq.args(), _ptr(codes), _ptr(ids), n, _ptr(queries), nq, STRATEGIES[strategy],
                                      k, tau, threads, _ptr(oi), _ptr(osc), _ptr(oc), _ptr(sv)))
    return oi, osc, oc, sv


def ref_buggy_topk(scores, ids, k):
    scores = np.ascontiguousarray(scores, np.float32)
    ids = np.ascontiguousarray(ids, np.int64)
    oi = np.empty(max(k, 1), np.int64)
    osc = np.empty(max(k, 1), np.float32)
    n = ref().ref_buggy_topk(_ptr(scores), _ptr(ids), scores.shape[0], k, _ptr(oi), _ptr(osc))
    return oi[:n], osc[:n]


# --------------------------------------------------------------------------- IVF
class IVFLists:
    """CSR inverted lists: cell c holds rows off[c]:off[c+1] of codes/ids."""

    def __init__(self, off, codes, ids):
        self.off = np.ascontiguousarray(off, np.uint64)
        self.codes = np.ascontiguousarray(codes, np.uint8)
        self.ids = np.ascontiguousarray(ids, np.int64)


def ivf_assign(x, centroids, threads=8):
    """Nearest coarse cell by sq_l2 (strict <, ties -> lowest cell)."""
    x = np.ascontiguousarray(x, np.float32)
    centroids = np.ascontiguousarray(centroids, np.float32)
    out = np.empty(x.shape[0], np.uint32)
    lib().po_ivf_assign(_ptr(x), x.shape[0], x.shape[1], _ptr(centroids), centroids.shape[0], threads, _ptr(out))
    return out


def ivf_build(pq: PQ, x, centroids, ids=None, assign=None):
    """Lists of residual codes encode(x - c_assign), grouped by cell, stable in input order."""
    x = np.ascontiguousarray(x, np.float32)
    centroids = np.ascontiguousarray(centroids, np.float32)
    n = x.shape[0]
    ids = np.arange(n, dtype=np.int64) if ids is None else np.asarray(ids, np.int64)
    assign = ivf_assign(x, centroids) if assign is None else np.ascontiguousarray(assign, np.uint32)
    codes = np.empty((n, pq.code_bytes), np.uint8)
    lib().po_ivf_encode_residuals(*pq.args(), _ptr(x), n, _ptr(centroids), _ptr(assign), _ptr(codes))
    order = np.argsort(assign, kind="stable")
    off = np.zeros(centroids.shape[0] + 1, np.uint64)
    off[1:] = np.cumsum(np.bincount(assign, minlength=centroids.shape[0]))
    return IVFLists(off, codes[order], ids[order]), assign


def ivf_search(pq: PQ, centroids, lists: IVFLists, queries, k, nprobe, tau=None, strategy="dual", cap=0, threads=8,
               return_hash=False):
    """search_coarse.  Returns ids, scores, counts, survivors, scanned, probes
    (+ the per-query survivor hash, sum of mix64(id), with return_hash)."""
    centroids = np.ascontiguousarray(centroids, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    nq = queries.shape[0]
    tau = pq.code_bits if tau is None else tau
    oi = np.empty((nq, k), np.int64)
    osc = np.empty((nq, k), np.float32)
    oc = np.empty(nq, np.uint32)
    sv = np.empty(nq, np.uint64)
    sc = np.empty(nq, np.uint64)
    pr = np.empty((nq, nprobe), np.uint32)
    sh = np.empty(nq, np.uint64)
    rc = lib().po_ivf_search(*pq.args(), _ptr(pq.inv_perms), _ptr(centroids), centroids.shape[0], _ptr(lists.off),
                             _ptr(lists.codes), _ptr(lists.ids), _ptr(queries), nq, nprobe, cap, STRATEGIES[strategy],
                             k, tau, threads, _ptr(oi), _ptr(osc), _ptr(oc), _ptr(sv), _ptr(sc), _ptr(pr), _ptr(sh))
    if rc != 0:
        raise ValueError(f"oracle ivf search rejected arguments (rc={rc})")
    if return_hash:
        return oi, osc, oc, sv, sc, pr, sh
    return oi, osc, oc, sv, sc, pr


def ref_kmeans(data, k, iters=25, seed=1234567):
    data = np.ascontiguousarray(data, np.float32)
    out = np.empty((k, data.shape[1]), np.float32)
    _check_ref(ref().ref_kmeans(_ptr(data), data.shape[0], data.shape[1], k, iters, seed, _ptr(out)))
    return out


def ref_assign_nearest(x, y):
    x = np.ascontiguousarray(x, np.float32)
    y = np.ascontiguousarray(y, np.float32)
    out = np.empty(x.shape[0], np.uint32)
    _check_ref(ref().ref_assign_nearest(_ptr(x), x.shape[0], _ptr(y), y.shape[0], x.shape[1], _ptr(out)))
    return out


def ref_ivf_search(pq: PQ, centroids, lists: IVFLists, queries, k, nprobe, tau=None, strategy="dual", cap=0,
                   threads=0):
    centroids = np.ascontiguousarray(centroids, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    nq = queries.shape[0]
    tau = pq.code_bits if tau is None else tau
    oi = np.empty((nq, k), np.int64)
    osc = np.empty((nq, k), np.float32)
    oc = np.empty(nq, np.uint32)
    sv = np.empty(nq, np.uint64)
    _check_ref(ref().ref_ivf_search(*pq.args(), _ptr(centroids), centroids.shape[0], _ptr(lists.off),
                                    _ptr(lists.codes), _ptr(lists.ids), _ptr(queries), nq, nprobe, cap,
                                    STRATEGIES[strategy], k, tau, threads, _ptr(oi), _ptr(osc), _ptr(oc), _ptr(sv)))
    return oi, osc, oc, sv


# ---------------------------------------------------------------- k-means (train_coarse)
class MT19937_64:
    """std::mt19937_64 (the engine of poly::Rng, common.hpp:45-67), in Python for the k-means
    restatement; pinned by the C++ standard's check value (10000th output of the default
    seed 5489 = 9981545732273789042, tests/test_kmeans_oracle.py)."""
    _M = (1 << 64) - 1

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & self._M
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & self._M
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & self._M

    def u01(self) -> float:  # Rng::u01 (common.hpp:51)
        return (self() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:  # Rng::below (common.hpp:55-63)
        if n <= 1:
            return 0
        limit = self._M - self._M % n
        while True:
            x = self()
            if x < limit:
                return x % n


def _sq_l2_rows(x, c):
    """sq_l2 (distances.cpp:10-17) of every row of x to c: fp32, dimension order, no FMA."""
    acc = np.zeros(x.shape[0], np.float32)
    for d in range(x.shape[1]):
        t = x[:, d] - c[d]
        acc = acc + t * t
    return acc


def _nearest_exact(x, cent):
    """assign_nearest (distances.cpp:56-79) with exact fp32 sq_l2, ties to the lower cell."""
    best = _sq_l2_rows(x, cent[0])
    arg = np.zeros(x.shape[0], np.uint32)
    for c in range(1, cent.shape[0]):
        d = _sq_l2_rows(x, cent[c])
        m = d < best
        best = np.where(m, d, best)
        arg[m] = c
    return arg, best


def kmeans_restated(data, k, iters=25, seed=1234567):
    """kmeans (kmeans.cpp:14-137) restated in numpy with the exact assignment the GPU uses
    (the reference's own assign_nearest goes through a BLAS GEMM).  Returns centroids,
    assign, iteration_mse, mse.  Small inputs only (O(n k d) numpy passes)."""
    x = np.ascontiguousarray(data, np.float32)
    n, dim = x.shape
    if n <= k:
        cent = np.stack([x[c % n] for c in range(k)])
        return cent, np.arange(n, dtype=np.uint32), [], 0.0
    rng = MT19937_64(seed)
    cent = np.empty((k, dim), np.float32)
    cent[0] = x[rng.below(n)]
    min_d2 = _sq_l2_rows(x, cent[0]).astype(np.float64)
    for c in range(1, k):
        total = float(np.sum(min_d2))  # (the reference sums sequentially; rounding may differ)
        if total <= 0.0:
            pick = rng.below(n)
        else:
            target = rng.u01() * total
            cs = np.cumsum(min_d2)
            hit = np.nonzero(target - cs <= 0.0)[0]
            pick = int(hit[0]) if hit.size else n - 1
        cent[c] = x[pick]
        min_d2 = np.minimum(min_d2, _sq_l2_rows(x, cent[c]).astype(np.float64))
    it_mse = []
    for _ in range(iters):
        assign, best = _nearest_exact(x, cent)
        it_mse.append(float(np.sum(best.astype(np.float64))) / n)
        counts = np.bincount(assign, minlength=k)
        sums = np.zeros((k, dim), np.float64)
        np.add.at(sums, assign, x.astype(np.float64))
        for c in range(k):
            if counts[c]:
                cent[c] = (sums[c] * (1.0 / counts[c])).astype(np.float32)
        for c in range(k):
            if counts[c]:
                continue
            big = int(np.argmax(counts))
            if counts[big] == 0:
                break
            members = np.nonzero(assign == big)[0]
            d = _sq_l2_rows(x[members], cent[big])
            far = int(members[int(np.argmax(d))])
            cent[c] = x[far]
            assign[far] = c
            counts[c] = 1
            counts[big] -= 1
    assign, best = _nearest_exact(x, cent)
    return cent, assign, it_mse, float(np.sum(best.astype(np.float64))) / n
