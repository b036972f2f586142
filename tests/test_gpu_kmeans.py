"""GPU k-means (poly_b200_kmeans, train_coarse SPEC.md:365-369; kmeans.cpp:14-137) against
the numpy restatement with the same exact assignment (oracle.kmeans_restated): the same
k-means++ picks (reference Rng draws), assignments and per-iteration objectives; centroids
to fp32 rounding (double sums in atomic order).  Also against the reference library's own
kmeans (BLAS assignment: near-ties may flip, so the objective is compared), the n <= k and
duplicate-point (empty cell) paths, and an IVF built on trained centroids."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1609_01882_b200 as pb
    return pb


@pytest.mark.parametrize("dim,n,k,iters", [(128, 20000, 64, 5), (40, 5000, 32, 3), (256, 8000, 300, 2)])
def test_kmeans_matches_restatement(pb, dim, n, k, iters):
    seed = 160901882
    centers = oracle.gen_centers(seed, 100, dim)
    x = oracle.gen_points(seed, 1, 0, n, centers)
    cent, assign, it_mse, mse = pb.kmeans(x, k, iters=iters, seed=7)
    rc, ra, rit, rmse = oracle.kmeans_restated(x, k, iters=iters, seed=7)
    assert np.array_equal(assign, ra)
    np.testing.assert_allclose(cent, rc, rtol=2e-6, atol=1e-6)
    np.testing.assert_allclose(it_mse, rit, rtol=1e-9)
    assert abs(mse - rmse) <= 1e-9 * rmse


def test_kmeans_close_to_reference_library(pb):
    if not oracle.ref_available():
        pytest.skip("reference library not built")
    seed = 160901882
    centers = oracle.gen_centers(seed, 100, 128)
    x = oracle.gen_points(seed, 1, 0, 10000, centers)
    cent, assign, _, mse = pb.kmeans(x, 50, iters=10, seed=1234567)
    ref = oracle.ref_kmeans(x, 50, iters=10, seed=1234567)
    a_ref = oracle.ref_assign_nearest(x, ref)
    d = ((x.astype(np.float64) - ref[a_ref]) ** 2).sum(1).mean()
    assert mse <= d * 1.01 and d <= mse * 1.01
    # most centroids coincide (the seeding draws are the reference's own)
    close = np.isclose(cent, ref, rtol=1e-4, atol=1e-4).all(1).mean()
    assert close >= 0.8, close


def test_kmeans_small_and_duplicates(pb):
    x = np.arange(12, dtype=np.float32).reshape(3, 4)
    cent, assign, it_mse, mse = pb.kmeans(x, 5)
    assert np.array_equal(cent[:3], x) and np.array_equal(cent[3:], x[:2]) and mse == 0.0
    assert np.array_equal(assign, [0, 1, 2])
    # 10 distinct points repeated: k = 20 leaves cells empty; stealing stops at singletons
    base = np.random.default_rng(1).normal(size=(10, 32)).astype(np.float32)
    xd = np.repeat(base, 50, axis=0)
    cent, assign, _, mse = pb.kmeans(xd, 20, iters=4, seed=3)
    rc, ra, _, rmse = oracle.kmeans_restated(xd, 20, iters=4, seed=3)
    assert np.array_equal(assign, ra) and mse == pytest.approx(rmse, abs=1e-9)
    with pytest.raises(pb.PolyError):
        pb.kmeans(np.zeros((0, 8), np.float32), 4)


def test_ivf_on_trained_coarse(pb, gi=None):
    """train_coarse -> build -> search_coarse: the GPU-trained quantizer in an IVF index
    gives the oracle's search results on the same lists."""
    import os
    seed = 160901882
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_ivf.npz"))
    pq = oracle.PQ(8, 8, 128, z["codebooks"], z["perms"])
    centers = oracle.gen_centers(seed, 1000, 128)
    train = oracle.gen_points(seed, 1, 0, 20000, centers)
    coarse, _, _, _ = pb.kmeans(train, 128, iters=8, seed=11)
    base = oracle.gen_points(seed, 2, 0, 100_000, centers)
    ix = pb.IVFIndex(pb.ProductQuantizer(8, 8, 128, z["codebooks"], z["perms"]), coarse)
    ix.add(base)
    lists, _ = oracle.ivf_build(pq, base, coarse)
    q = oracle.gen_points(seed, 3, 0, 200, centers)
    oi, osc, oc, _, _, _ = oracle.ivf_search(pq, coarse, lists, q, 50, 16, tau=26, threads=16)
    ids, sc, cnt = ix.search(q, pb.CoarseParams(pb.Strategy.dual, 50, 26, 16, 0))
    assert np.array_equal(ids, oi) and np.array_equal(cnt, oc)
    assert np.array_equal(sc.view(np.uint32), osc.view(np.uint32))
