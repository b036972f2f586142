"""The k-means restatement (oracle.kmeans_restated, kmeans.cpp:14-137) and its RNG: the
Python mt19937_64 against the C++ standard's check value, Rng::u01 / below semantics,
and the restatement's invariants on a small mixture (objective non-increasing, every
point assigned to its exact nearest centroid, centroids = member means).  CPU only."""
import numpy as np

import oracle


def test_mt19937_64_check_value():
    g = oracle.MT19937_64(5489)
    for _ in range(9999):
        g()
    assert g() == 9981545732273789042  # [rand.predef]: the 10000th invocation


def test_rng_helpers():
    g = oracle.MT19937_64(1234567)
    u = [g.u01() for _ in range(1000)]
    assert all(0.0 <= v < 1.0 for v in u)
    b = [g.below(7) for _ in range(1000)]
    assert set(b) == set(range(7))
    assert oracle.MT19937_64(3).below(1) == 0


def test_restated_kmeans_invariants():
    seed = 160901882
    centers = oracle.gen_centers(seed, 50, 32)
    x = oracle.gen_points(seed, 1, 0, 3000, centers)
    cent, assign, it_mse, mse = oracle.kmeans_restated(x, 40, iters=6, seed=7)
    assert len(it_mse) == 6
    assert all(b <= a * (1 + 1e-12) for a, b in zip(it_mse, it_mse[1:] + [mse]))
    d = ((x[:, None, :].astype(np.float64) - cent[None, :, :]) ** 2).sum(-1)
    assert (d[np.arange(len(x)), assign] <= d.min(1) * (1 + 1e-5) + 1e-6).all()
    assert len(np.unique(assign)) == 40  # no empty cell with n >> k distinct points


def test_small_n_replicates_points():
    x = np.arange(12, dtype=np.float32).reshape(3, 4)
    cent, assign, it_mse, mse = oracle.kmeans_restated(x, 5)
    assert np.array_equal(cent[:3], x) and np.array_equal(cent[3:], x[:2]) and mse == 0.0
