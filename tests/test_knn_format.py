"""The k-NN graph file format (knn_format.py, written by poly_b200_knn_writer_*): reference
writer -> reader round trip, and the reader's error classes (poly::errc: format, version,
corrupt) on damaged files.  CPU only."""
import numpy as np
import pytest

from paper_1609_01882_b200 import knn_format
from paper_1609_01882_b200.flat_index import Errc, PolyError


def _rows(n=40, k=6, seed=3):
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, k + 1, n).astype(np.uint32)
    nbr = np.full((n, k), -1, np.int64)
    sc = np.full((n, k), np.inf, np.float32)
    for i in range(n):
        nbr[i, :counts[i]] = rng.integers(-2**40, 2**40, counts[i])
        sc[i, :counts[i]] = np.sort(rng.random(counts[i]).astype(np.float32))
    return np.arange(100, 100 + n), counts, nbr, sc


def test_round_trip(tmp_path):
    ids, counts, nbr, sc = _rows()
    p = tmp_path / "g.knng"
    knn_format.write_graph(p, 6, ids, counts, nbr, sc)
    k, rid, rc, rn, rs = knn_format.read_graph(p)
    assert k == 6 and np.array_equal(rid, ids) and np.array_equal(rc, counts)
    assert np.array_equal(rn, nbr) and np.array_equal(rs.view(np.uint32), sc.view(np.uint32))


def test_empty_graph(tmp_path):
    p = tmp_path / "e.knng"
    knn_format.write_graph(p, 3, [], [], [], [])
    k, rid, rc, rn, rs = knn_format.read_graph(p)
    assert k == 3 and rid.size == 0 and rn.shape == (0, 3)


@pytest.mark.parametrize("where,code", [(0, Errc.format), (8, Errc.version), (60, Errc.corrupt)])
def test_damage_is_detected(tmp_path, where, code):
    ids, counts, nbr, sc = _rows()
    p = tmp_path / "g.knng"
    knn_format.write_graph(p, 6, ids, counts, nbr, sc)
    b = bytearray(p.read_bytes())
    b[where] ^= 0x5A
    p.write_bytes(bytes(b))
    with pytest.raises(PolyError) as e:
        knn_format.read_graph(p)
    assert e.value.code == code


def test_truncated(tmp_path):
    ids, counts, nbr, sc = _rows()
    p = tmp_path / "g.knng"
    knn_format.write_graph(p, 6, ids, counts, nbr, sc)
    p.write_bytes(p.read_bytes()[:-7])
    with pytest.raises(PolyError) as e:
        knn_format.read_graph(p)
    assert e.value.code == Errc.corrupt
