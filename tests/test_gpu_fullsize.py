"""Parity at BASELINE.json sizes through size-independent properties plus a
seeded random subset checked against the CPU oracle (which is bitwise the
reference, tests/test_oracle.py)."""

import numpy as np
import pytest

from oracle import mps_oracle as O

pytestmark = pytest.mark.gpu

CONFIGS = {
    # name: (m, d, gamma, budget, N_train, N_test, tolerance)
    "headline_m165_d1": (165, 1, 0.1, 1e-24, 6400, 1600, 1e-10),
    "config2_m50_d2": (50, 2, 0.1, 1e-24, 800, 200, 1e-10),
    "config3_m100_d4": (100, 4, 0.1, 1e-16, 1600, 400, 1e-6),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_full_size_kernel_properties_and_oracle_subset(name):
    import paper_2411_09336_b200 as P

    m, d, gamma, budget, n, mt, tol = CONFIGS[name]
    cfg = P.FeatureMapConfig(m, 2, d, gamma)
    X = np.random.default_rng(0).uniform(0.0, 2.0, (n, m))
    Xt = np.random.default_rng(1).uniform(0.0, 2.0, (mt, m))
    tr = P.simulate_dataset(X, cfg, budget=budget)
    te = P.simulate_dataset(Xt, cfg, budget=budget)
    K = P.compute_gram(tr, tr, "train").entries
    Kt = P.compute_gram(te, tr, "test").entries
    # size-independent properties (acceptance C5)
    assert np.array_equal(K, K.T)
    assert np.all(np.diag(K) == 1.0)
    assert K.min() >= 0.0 and K.max() <= 1.0 + 1e-12
    assert Kt.min() >= 0.0 and Kt.max() <= 1.0 + 1e-12
    if name.startswith("headline"):
        assert tr.bond_dims().max() <= 4  # acceptance C6's resource claim
    # random subset against the oracle
    rng = np.random.default_rng(123)
    idx = np.sort(rng.choice(n, 8, replace=False))
    tidx = np.sort(rng.choice(mt, 3, replace=False))
    ref = [O.simulate_row(X[i], m, 2, d, gamma, budget) for i in idx]
    reft = [O.simulate_row(Xt[i], m, 2, d, gamma, budget) for i in tidx]
    chi = tr.bond_dims()
    mismatches = sum(chi[i].tolist() != r.bond_dims() for i, r in zip(idx, ref))
    assert mismatches == 0, f"{mismatches} of {len(idx)} states differ in bond dims"
    Ko = O.gram([r.sites for r in ref], [r.sites for r in ref], "train")
    assert np.abs(K[np.ix_(idx, idx)] - Ko).max() < tol
    Kto = O.gram([r.sites for r in reft], [r.sites for r in ref], "test")
    assert np.abs(Kt[np.ix_(tidx, idx)] - Kto).max() < tol
