"""The inverted-list file layout (paper_1609_01882_b200/ivf_format.py restates what
poly_b200_ivf_save / _load implement in csrc/capi_ivf.cu): round trip and the poly::errc
classes of damaged files (common.hpp:13-22: format, version, corrupt).  CPU only; the
GPU tests (test_gpu_ivf_io.py) cross the C++ writer with this reader and back."""
import os
import struct
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_1609_01882_b200"))
import ivf_format as F  # noqa: E402  (the module needs no GPU; the package import would load the CUDA library)


def _sample(rng, m=8, nlist=7, n=300):
    dim = 16 * m
    cells = rng.integers(0, nlist, n)
    off = np.zeros(nlist + 1, np.uint64)
    off[1:] = np.cumsum(np.bincount(cells, minlength=nlist))
    return (m, dim, rng.normal(size=(m, 256, 16)).astype(np.float32),
            np.stack([rng.permutation(256) for _ in range(m)]).astype(np.uint16),
            rng.normal(size=(nlist, dim)).astype(np.float32), off,
            rng.integers(0, 256, (n, m)).astype(np.uint8), rng.permutation(n).astype(np.int64) * 3 + 5)


@pytest.mark.parametrize("m", [8, 16])
def test_round_trip(tmp_path, m):
    t = _sample(np.random.default_rng(m), m=m)
    p = tmp_path / "lists.ivf"
    F.write(p, *t)
    got = F.read(p)
    for a, b in zip(t, got):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    m2, dim2, cb, perms, coarse = F.read_header_tables(p)
    assert (m2, dim2) == (m, 16 * m) and np.array_equal(coarse, t[4])


def test_damaged_files_map_to_errc(tmp_path):
    t = _sample(np.random.default_rng(3))
    p = tmp_path / "lists.ivf"
    F.write(p, *t)
    raw = bytearray(p.read_bytes())
    cases = {}
    bad = bytearray(raw); bad[0] ^= 1; cases["format"] = bad                        # magic
    bad = bytearray(raw); bad[8:12] = struct.pack("<I", 2); cases["version"] = bad   # version
    bad = bytearray(raw); bad[-5] ^= 0x40; cases["corrupt"] = bad                    # id payload bit flip
    for errc, data in cases.items():
        q = tmp_path / f"{errc}.ivf"
        q.write_bytes(bytes(data))
        with pytest.raises(F.FormatError) as e:
            F.read(q)
        assert e.value.errc == errc
    q = tmp_path / "short.ivf"
    q.write_bytes(bytes(raw[:len(raw) // 2]))
    with pytest.raises(F.FormatError) as e:
        F.read(q)
    assert e.value.errc == "corrupt"
