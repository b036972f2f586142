"""Pin the IVF restatement (oracle po_ivf_*) to golden vectors composed from
the reference's primitives (tests/golden/golden_ivf.npz)."""
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_ivf.npz")


@pytest.fixture(scope="module")
def gi():
    z = dict(np.load(GOLDEN))
    z["pq"] = oracle.PQ(8, 8, 128, z["codebooks"], z["perms"])
    z["lists"] = oracle.IVFLists(z["off"], z["list_codes"], z["list_ids"])
    return z


def test_build_matches_reference(gi):
    centers = oracle.gen_centers(int(gi["data_seed"]), 1000, 128)
    base = oracle.gen_points(int(gi["data_seed"]), 2, 0, int(gi["n"]), centers)
    assert np.array_equal(base[:64], gi["base_head"])
    assign = oracle.ivf_assign(base, gi["coarse"])
    assert np.array_equal(assign, gi["assign_exact"])
    assert np.array_equal(assign, gi["assign_ref"])  # no near-tie flips vs the GEMM path on this data
    lists, _ = oracle.ivf_build(gi["pq"], base, gi["coarse"], ids=np.arange(int(gi["n"])) * 7 + 3, assign=assign)
    assert np.array_equal(lists.off, gi["off"])
    assert np.array_equal(lists.codes, gi["list_codes"])
    assert np.array_equal(lists.ids, gi["list_ids"])


@pytest.mark.parametrize("nprobe", [1, 4, 16, 64])
def test_search_coarse_matches_reference(gi, nprobe):
    for tau in (20, 26, 64):
        for cap in (0, 1500):
            key = f"p{nprobe}_t{tau}_c{cap}"
            i, s, c, sv, scanned, probes = oracle.ivf_search(gi["pq"], gi["coarse"], gi["lists"], gi["queries"], 50,
                                                             nprobe, tau=tau, cap=cap)
            assert np.array_equal(i, gi[key + "_ids"]), key
            assert np.array_equal(s.view(np.uint32), gi[key + "_scores"].view(np.uint32)), key
            assert np.array_equal(c, gi[key + "_counts"]), key
            assert np.array_equal(sv, gi[key + "_surv"]), key
            if cap:
                assert (scanned >= np.minimum(cap, scanned)).all()


def test_strategies_and_boundary(gi):
    for strat in ("adc", "binary"):
        i, s, c, _, _, _ = oracle.ivf_search(gi["pq"], gi["coarse"], gi["lists"], gi["queries"], 50, 16,
                                             strategy=strat)
        assert np.array_equal(i, gi[f"{strat}16_ids"])
        assert np.array_equal(s.view(np.uint32), gi[f"{strat}16_scores"].view(np.uint32))
    # all probes, no cap, tau = code_bits == exhaustive IVF-ADC over every list
    i, s, c, _, scanned, _ = oracle.ivf_search(gi["pq"], gi["coarse"], gi["lists"], gi["queries"], 50, 64, tau=64)
    assert (scanned == int(gi["n"])).all()
    assert np.array_equal(i, gi["p64_t64_c0_ids"])
    # probe monotonicity of the survivor sets: more probes, more survivors
    prev = None
    for nprobe in (1, 4, 16, 64):
        sv = gi[f"p{nprobe}_t26_c0_surv"]
        if prev is not None:
            assert (sv >= prev).all()
        prev = sv
