"""Pin the CPU restatement (oracle/polyoracle.c) to the reference's own outputs.

The golden vectors were produced by the reference's compiled sources
(tests/golden/make_golden.py -> oracle/_ref/libpolyref.so).  Every check is
bit-exact: integer/byte work and the fp32 LUT/ADC sums use the same operation
order as the reference.
"""
import numpy as np
import pytest

import oracle

TAUS8 = (0, 20, 24, 28, 32, 64)
TAUS16 = (0, 48, 56, 64, 128)


def _gen_inputs(pq, g, normalize=False):
    centers = oracle.gen_centers(int(g["data_seed"]), int(g["ncent"]), pq.dim)
    base = oracle.gen_points(int(g["data_seed"]), 2, 0, int(g["n"]), centers, normalize)
    queries = oracle.gen_points(int(g["data_seed"]), 3, 0, g["queries"].shape[0], centers, normalize)
    return base, queries


@pytest.mark.parametrize("which", ["8", "16"])
def test_generator_reproduces_fixture_inputs(which, pq8, pq16, g8, g16):
    pq, g = (pq8, g8) if which == "8" else (pq16, g16)
    base, queries = _gen_inputs(pq, g)
    assert np.array_equal(base[:64], g["base_head"])
    assert np.array_equal(queries, g["queries"])


@pytest.mark.parametrize("which", ["8", "16"])
def test_encode_lut_bit_exact(which, pq8, pq16, g8, g16):
    pq, g = (pq8, g8) if which == "8" else (pq16, g16)
    base, queries = _gen_inputs(pq, g)
    assert np.array_equal(oracle.encode(pq, base), g["codes"])           # pq.cpp:29-45
    lut, lutp, qc = oracle.lut_batch(pq, queries)
    assert np.array_equal(qc, g["qcodes"])
    assert np.array_equal(lut[:4].view(np.uint32), g["lut"].view(np.uint32))   # pq.cpp:91-105
    assert np.array_equal(lutp[:4].view(np.uint32), g["lutp"].view(np.uint32)) # pq.cpp:107-119
    # query code == perm[argmin LUT row]
    am = lut.argmin(axis=2)
    for sq in range(pq.m):
        assert np.array_equal(qc[:, sq], pq.perms[sq][am[:, sq]].astype(np.uint8))


@pytest.mark.parametrize("which", ["8", "16"])
def test_hamming_and_adc_matrices(which, pq8, pq16, g8, g16):
    pq, g = (pq8, g8) if which == "8" else (pq16, g16)
    qc, codes = g["qcodes"], g["codes"][:2000]
    ham = np.array([[oracle.hamming(a, b) for b in codes[:300]] for a in qc[:6]])
    assert np.array_equal(ham, g["ham"][:6, :300])
    # ADC via the permuted table == adc_distance (pq.cpp:121-128), bit-exact
    lutp = g["lutp"]
    adc = np.zeros((4, 2000), np.float32)
    for sq in range(pq.m):
        adc = adc + lutp[:, sq, :][:, codes[:, sq]]
    assert np.array_equal(adc.view(np.uint32), g["adc"].view(np.uint32))


@pytest.mark.parametrize("strategy", ["adc", "binary", "disidx"])
@pytest.mark.parametrize("which", ["8", "16"])
def test_search_strategies_match_reference(strategy, which, pq8, pq16, g8, g16):
    pq, g = (pq8, g8) if which == "8" else (pq16, g16)
    i, s, c, _, _ = oracle.search(pq, g["codes"], g["queries"], 100, strategy=strategy)
    assert np.array_equal(i, g[f"{strategy}_ids"])
    assert np.array_equal(s.view(np.uint32), g[f"{strategy}_scores"].view(np.uint32))
    assert np.array_equal(c, g[f"{strategy}_counts"])


@pytest.mark.parametrize("which", ["8", "16"])
def test_dual_search_matches_reference(which, pq8, pq16, g8, g16):
    pq, g, taus = (pq8, g8, TAUS8) if which == "8" else (pq16, g16, TAUS16)
    for tau in taus:
        i, s, c, sv, _ = oracle.search(pq, g["codes"], g["queries"], 100, tau=tau)
        assert np.array_equal(i, g[f"dual{tau}_ids"]), tau
        assert np.array_equal(s.view(np.uint32), g[f"dual{tau}_scores"].view(np.uint32)), tau
        assert np.array_equal(c, g[f"dual{tau}_counts"]), tau
        assert np.array_equal(sv, g[f"dual{tau}_surv"]), tau
    # dual at tau = code_bits is adc, id for id
    assert np.array_equal(g[f"dual{pq.code_bits}_ids"], g["adc_ids"])


@pytest.mark.parametrize("which", ["8", "16"])
def test_ties_and_shortage(which, pq8, pq16, g8, g16):
    pq, g, taus = (pq8, g8, TAUS8) if which == "8" else (pq16, g16, TAUS16)
    tie_codes = np.repeat(g["codes"][:500], 4, axis=0)
    for tau in (taus[1], pq.code_bits):
        i, s, c, sv, _ = oracle.search(pq, tie_codes, g["queries"], 7, tau=tau, ids=g["tie_ids_in"])
        assert np.array_equal(i, g[f"tie{tau}_ids"])
        assert np.array_equal(c, g[f"tie{tau}_counts"])
        assert np.array_equal(sv, g[f"tie{tau}_surv"])
        # ties broken by lower id
        for r in range(i.shape[0]):
            n = c[r]
            key = list(zip(s[r, :n].tolist(), i[r, :n].tolist()))
            assert key == sorted(key)


def test_topk_contract_vs_reference_defect():
    z = np.load(oracle.__file__.replace("__init__.py", "../tests/golden/topk_kat.npz"))
    # the reference TopK (flat_index.hpp:60-94) returned {1, 5}; the contract is {1, 3}
    assert z["buggy_scores"].tolist() == [1.0, 5.0]
    ids, sc = oracle.topk_select(z["offers"], np.arange(4), 2)
    assert sc.tolist() == [1.0, 3.0] and ids.tolist() == [3, 1]
    assert float(z["buggy_mismatch_rate"]) > 0.3
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = int(rng.integers(0, 80))
        s = rng.integers(0, 10, n).astype(np.float32)
        ii = rng.permutation(n).astype(np.int64) * 5
        k = int(rng.integers(0, 15))
        gi, gs = oracle.topk_select(s, ii, k)
        want = sorted(zip(s.tolist(), ii.tolist()))[:k]
        assert list(zip(gs.tolist(), gi.tolist())) == want


def test_edge_cases(pq8, g8):
    q = g8["queries"][:3]
    i, s, c, sv, _ = oracle.search(pq8, g8["codes"], q, 0, tau=24)           # k = 0 -> empty
    assert c.tolist() == [0, 0, 0]
    i, s, c, sv, _ = oracle.search(pq8, g8["codes"][:0], q, 10, tau=24)      # empty index -> empty
    assert c.tolist() == [0, 0, 0] and (i == -1).all() and np.isinf(s).all()
    with pytest.raises(ValueError):
        oracle.search(pq8, g8["codes"], q, 10, tau=65)                      # tau > code_bits


def test_calibrate_and_relabel(pq8, g8):
    codes, q = g8["codes"], g8["queries"]
    tau, warn = oracle.calibrate_threshold(pq8, codes, q, 0.95)
    hist = oracle.hamming_histogram(pq8, codes, q)
    frac = hist.cumsum(axis=1).mean(axis=0) / codes.shape[0]
    assert not warn and frac[tau] <= 0.05 and (tau == 64 or frac[tau + 1] > 0.05)
    # flat_index.hpp:128-130: max{tau : mean survivor fraction <= 1 - rate}
    for rate in (1e-9, 0.5, 0.8, 0.99):
        t, w = oracle.calibrate_threshold(pq8, codes, q, rate)
        ok = np.nonzero(frac <= 1.0 - rate)[0]
        assert (t, w) == ((int(ok.max()), False) if ok.size else (0, True))
    # relabel to identity assignments == encoding with an identity-perm PQ
    ident = np.tile(np.arange(256, dtype=np.uint16), (8, 1))
    pq_id = oracle.PQ(8, 8, 128, pq8.codebooks, ident)
    base = oracle.gen_points(int(g8["data_seed"]), 2, 0, 500, oracle.gen_centers(int(g8["data_seed"]), 1000, 128))
    assert np.array_equal(oracle.relabel_codes(pq8, ident, codes[:500]), oracle.encode(pq_id, base))
