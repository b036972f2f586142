"""Seeded Gaussian-mixture workload generator (host side, numpy).

Bit-identical to csrc/synth.cuh (device) and oracle/polyoracle.c (checker):
splitmix64 hashing in wrapping uint64 arithmetic, Irwin-Hall(12) normals via
an exact int64 -> fp32 conversion, fp32 adds/muls.  The large database is
generated on the GPU by ``FlatIndex.add_synthetic``; this module produces the
small pieces the host needs (mixture centers, query rows).

BASELINE.json configs: centers ~ N(0,1) * 10, points = max(0, center + N(0,1)).
Stream ids: 0 centers, 1 train, 2 base, 3 queries.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z):
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _row_keys(seed, stream, rows):
    with np.errstate(over="ignore"):
        base = _mix64(np.uint64(seed) + np.uint64(0x632BE59BD9B4E019) * np.uint64(stream + 1))
        return _mix64(base ^ (rows.astype(np.uint64) * np.uint64(0xD1B54A32D192ED03)))


def _normals(keys, dim):
    """keys [n] -> N(0,1) approximations [n, dim] (Irwin-Hall of 12 24-bit uniforms)."""
    t = np.arange(dim, dtype=np.uint64)
    s = np.zeros((keys.shape[0], dim), np.uint64)
    with np.errstate(over="ignore"):
        for j in range(6):
            salt = (np.uint64(6) * t + np.uint64(j + 1)) * np.uint64(0xA0761D6478BD642F)
            h = _mix64(keys[:, None] ^ salt[None, :])
            s += (h >> np.uint64(40)) + ((h >> np.uint64(16)) & np.uint64(0xFFFFFF))
    c = s.astype(np.int64) - np.int64(6 * 16777216)
    return c.astype(np.float32) * np.float32(1.0 / 16777216.0)


def gen_centers(seed: int, ncent: int, dim: int) -> np.ndarray:
    keys = _row_keys(seed, 0, np.arange(ncent, dtype=np.uint64))
    return (np.float32(10.0) * _normals(keys, dim)).astype(np.float32)


def gen_points(seed: int, stream: int, row0: int, n: int, centers: np.ndarray, normalize: bool = False):
    ncent, dim = centers.shape
    keys = _row_keys(seed, stream, np.arange(row0, row0 + n, dtype=np.uint64))
    with np.errstate(over="ignore"):
        u = (((_mix64(keys ^ np.uint64(0x5851F42D4C957F2D)) >> np.uint64(32)) * np.uint64(ncent)) >> np.uint64(32))
    x = centers[u.astype(np.int64)] + _normals(keys, dim)
    x = np.where(x > 0, x, np.float32(0)).astype(np.float32)
    if normalize:
        nrm = np.zeros(n, np.float32)
        for t in range(dim):  # sequential fp32 accumulation, as the oracle / GPU do
            nrm = (nrm + x[:, t] * x[:, t]).astype(np.float32)
        inv = np.where(nrm > 0, np.float32(1.0) / np.sqrt(nrm), np.float32(0)).astype(np.float32)
        x = (x * inv[:, None]).astype(np.float32)
    return x
