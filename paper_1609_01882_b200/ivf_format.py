"""The inverted-list file written by poly_b200_ivf_save / read by poly_b200_ivf_load
(csrc/capi_ivf.cu), restated in numpy: the layout reference for other readers and the
CPU-side check of the format.  Little-endian throughout.

    header   char magic[8] = "POLYIVF\\0"; u32 version = 1; u32 m; u32 dbits = 8;
             u32 dim; u32 nlist; u32 0; u64 n
    sections char tag[8]; u64 bytes; u64 fnv1a64(payload); payload -- in this order:
             PQCODEBK  m x 256 x (dim / m) fp32   codebooks (pq.hpp:52)
             PQPERMS_  m x 256 u16                 perms: centroid -> stored field (pq.hpp:54)
             COARSE__  nlist x dim fp32            coarse centroids
             LISTOFF_  (nlist + 1) u64             CSR offsets: cell c holds rows off[c]:off[c+1]
             CODES___  n x m u8                    residual codes, list order
             IDS_____  n i64                       ids, list order

Errors (poly::errc, common.hpp:13-22): io (open / write), format (magic, section tag or
size, shape), version, corrupt (checksum, truncation, offsets).
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"POLYIVF\0"
VERSION = 1
TAGS = (b"PQCODEBK", b"PQPERMS_", b"COARSE__", b"LISTOFF_", b"CODES___", b"IDS_____")


class FormatError(ValueError):
    def __init__(self, errc: str, msg: str):
        super().__init__(msg)
        self.errc = errc  # "io" | "format" | "version" | "corrupt"


def fnv1a64(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    a = np.frombuffer(data, np.uint8)
    h = np.uint64(h)
    prime = np.uint64(0x100000001B3)
    with np.errstate(over="ignore"):
        for b in a:  # byte loop: for test-sized files only
            h = (h ^ np.uint64(b)) * prime
    return int(h)


def write(path, m, dim, codebooks, perms, coarse, off, codes, ids):
    codebooks = np.ascontiguousarray(codebooks, "<f4")
    perms = np.ascontiguousarray(perms, "<u2")
    coarse = np.ascontiguousarray(coarse, "<f4")
    off = np.ascontiguousarray(off, "<u8")
    codes = np.ascontiguousarray(codes, np.uint8)
    ids = np.ascontiguousarray(ids, "<i8")
    nlist, n = coarse.shape[0], int(off[-1])
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<6I", VERSION, m, 8, dim, nlist, 0) + struct.pack("<Q", n))
        for tag, arr in zip(TAGS, (codebooks, perms, coarse, off, codes, ids)):
            b = arr.tobytes()
            f.write(tag + struct.pack("<QQ", len(b), fnv1a64(b)) + b)


def _sections(path, checksums=True, want=TAGS):
    with open(path, "rb") as f:
        head = f.read(40)
        if head[:8] != MAGIC:
            raise FormatError("format", "not an IVF list file (bad magic)")
        if len(head) < 40:
            raise FormatError("corrupt", "truncated IVF list file")
        version, m, dbits, dim, nlist, _ = struct.unpack_from("<6I", head, 8)
        (n,) = struct.unpack_from("<Q", head, 32)
        if version != VERSION:
            raise FormatError("version", f"unsupported IVF list file version {version}")
        out = {}
        for tag in TAGS:
            sh = f.read(24)
            if len(sh) < 24:
                raise FormatError("corrupt", "truncated IVF list file")
            if sh[:8] != tag:
                raise FormatError("format", f"expected section {tag.decode()}")
            nb, h = struct.unpack_from("<QQ", sh, 8)
            if tag not in want:
                f.seek(nb, 1)
                continue
            payload = f.read(nb)
            if len(payload) < nb:
                raise FormatError("corrupt", "truncated IVF list file")
            if checksums and fnv1a64(payload) != h:
                raise FormatError("corrupt", f"checksum mismatch in section {tag.decode()}")
            out[tag] = payload
    return (m, dbits, dim, nlist, n), out


def read(path, checksums=True):
    """(m, dim, codebooks, perms, coarse, off, codes, ids) -- raises FormatError."""
    (m, _, dim, nlist, n), s = _sections(path, checksums)
    codebooks = np.frombuffer(s[TAGS[0]], "<f4").reshape(m, 256, dim // m)
    perms = np.frombuffer(s[TAGS[1]], "<u2").reshape(m, 256)
    coarse = np.frombuffer(s[TAGS[2]], "<f4").reshape(nlist, dim)
    off = np.frombuffer(s[TAGS[3]], "<u8")
    codes = np.frombuffer(s[TAGS[4]], np.uint8).reshape(n, m)
    ids = np.frombuffer(s[TAGS[5]], "<i8")
    if off[0] != 0 or off[-1] != n or (np.diff(off.astype(np.int64)) < 0).any():
        raise FormatError("corrupt", "list offsets do not cover the codes")
    return m, dim, codebooks, perms, coarse, off, codes, ids


def read_header_tables(path):
    """(m, dim, codebooks, perms, coarse): the small sections only, unchecked."""
    (m, _, dim, nlist, _), s = _sections(path, checksums=False, want=TAGS[:3])
    return (m, dim, np.frombuffer(s[TAGS[0]], "<f4").reshape(m, 256, dim // m),
            np.frombuffer(s[TAGS[1]], "<u2").reshape(m, 256), np.frombuffer(s[TAGS[2]], "<f4").reshape(nlist, dim))
