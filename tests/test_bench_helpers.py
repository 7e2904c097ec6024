"""bench.py's roofline arithmetic: train_flops (prefix-sum form) equals the
direct sum of the per-pair algorithmic flop formula."""

import numpy as np

from oracle import mps_oracle as O


def test_train_flops_matches_direct_pair_sum():
    import bench

    rng = np.random.default_rng(0)
    chi = rng.integers(1, 5, size=(37, 12))
    chi[:, 0] = chi[:, -1] = 1
    direct = sum(O.overlap_flops(chi[i], chi[j]) for i in range(37) for j in range(i + 1, 37))
    assert bench.train_flops(chi) == float(direct)


def test_feature_rows_are_seeded_and_in_range():
    import bench

    X = bench.feature_rows(10, 7)
    assert X.shape == (10, 7) and X.min() >= 0.0 and X.max() <= 2.0
    assert np.array_equal(X, bench.feature_rows(10, 7))
