"""The k-NN graph file (External Interfaces: "one record per vector -- id,
neighbor count, then (neighbor id, score) pairs -- in a sectioned binary file plus an
optional ivecs export of neighbor ids"), as written by poly_b200_knn_writer_* (capi_ivf.cu).

    magic "POLYKNNG", u32 version (1), u32 k, u64 records,
    section { char tag[8] = "RECORDS_", u64 bytes, u64 fnv1a64(payload), payload }
    payload = records { i64 id, u32 count, count x { i64 neighbor id, f32 score } }, packed

all little-endian.  ivecs: per record an int32 k, then k int32 neighbor ids (-1 pads).
Pure numpy; read_graph checks the checksum and the record structure.
"""
from __future__ import annotations

import numpy as np

from .flat_index import Errc, PolyError

MAGIC = b"POLYKNNG"
VERSION = 1


def fnv1a64(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    b = np.frombuffer(data, np.uint8)
    for x in b.tolist():  # small files only (tests)
        h = ((h ^ x) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def write_graph(path, k: int, ids, counts, nbr_ids, scores):
    """Reference writer (tests): the same bytes the C ABI writes for these rows."""
    recs = bytearray()
    for i in range(len(ids)):
        c = int(counts[i])
        recs += np.int64(ids[i]).tobytes() + np.uint32(c).tobytes()
        for j in range(c):
            recs += np.int64(nbr_ids[i][j]).tobytes() + np.float32(scores[i][j]).tobytes()
    with open(path, "wb") as f:
        f.write(MAGIC + np.uint32(VERSION).tobytes() + np.uint32(k).tobytes() + np.uint64(len(ids)).tobytes())
        f.write(b"RECORDS_" + np.uint64(len(recs)).tobytes() + np.uint64(fnv1a64(bytes(recs))).tobytes())
        f.write(bytes(recs))


def read_graph(path, check_sum: bool = True):
    """Returns k, ids (n,), counts (n,), neighbor ids (n, k; -1 pads), scores (n, k; +inf pads)."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:8] != MAGIC:
        raise PolyError(Errc.format, "not a k-NN graph file (bad magic)")
    ver, k = np.frombuffer(raw, np.uint32, 2, 8)
    if ver != VERSION:
        raise PolyError(Errc.version, f"unsupported k-NN graph file version {ver}")
    n = int(np.frombuffer(raw, np.uint64, 1, 16)[0])
    if raw[24:32] != b"RECORDS_":
        raise PolyError(Errc.format, "expected section RECORDS_")
    nbytes, h = (int(x) for x in np.frombuffer(raw, np.uint64, 2, 32))
    payload = raw[48:48 + nbytes]
    if len(payload) != nbytes:
        raise PolyError(Errc.corrupt, "truncated k-NN graph file")
    if check_sum and fnv1a64(payload) != h:
        raise PolyError(Errc.corrupt, "checksum mismatch in section RECORDS_")
    k = int(k)
    ids = np.empty(n, np.int64)
    counts = np.empty(n, np.uint32)
    nbr = np.full((n, k), -1, np.int64)
    sc = np.full((n, k), np.inf, np.float32)
    at = 0
    for i in range(n):
        ids[i] = np.frombuffer(payload, np.int64, 1, at)[0]
        c = int(np.frombuffer(payload, np.uint32, 1, at + 8)[0])
        if c > k:
            raise PolyError(Errc.corrupt, "record with more than k neighbors")
        counts[i] = c
        rec = np.frombuffer(payload, np.dtype([("id", "<i8"), ("s", "<f4")]), c, at + 12)
        nbr[i, :c] = rec["id"]
        sc[i, :c] = rec["s"]
        at += 12 + 12 * c
    if at != nbytes:
        raise PolyError(Errc.corrupt, "record bytes do not add up to the section size")
    return k, ids, counts, nbr, sc


def read_ivecs(path):
    a = np.fromfile(path, np.int32)
    if a.size == 0:
        return np.zeros((0, 0), np.int32)
    d = int(a[0])
    return a.reshape(-1, d + 1)[:, 1:]
