"""The CPU oracle (oracle/mps_oracle.py) pinned against the golden fixtures
that tests/golden/make_golden.py recorded from the real reference."""

import numpy as np
import pytest

from conftest import golden, unpack_states
from oracle import mps_oracle as O


def _cfg(g):
    return int(g["m"]), int(g["r"]), int(g["d"]), float(g["gamma"]), float(g["budget"])


@pytest.mark.parametrize("name,n", [("config1_m8_d1.npz", 64), ("headline_m165_d1.npz", 6), ("config2_m50_d2.npz", 6)])
def test_oracle_states_match_reference_bitwise(name, n):
    g = golden(name)
    m, r, d, gamma, budget = _cfg(g)
    states = [O.simulate_row(x, m, r, d, gamma, budget) for x in g["X"][:n]]
    chi = np.array([s.bond_dims() for s in states])
    assert np.array_equal(chi, g["train_chi"][:n])
    assert np.array_equal([s.discard for s in states], g["train_discard"][:n])
    assert np.array_equal([s.peak for s in states], g["train_peak"][:n])
    K = O.gram([s.sites for s in states], [s.sites for s in states], "train")
    assert np.array_equal(K, g["K_train"][:n, :n])
    if "train_entries" in g:
        ref = unpack_states(g)
        for a, b in zip(states, ref):
            for x, y in zip(a.sites, b):
                assert np.array_equal(x, y)


def test_oracle_test_kernel_config1():
    g = golden("config1_m8_d1.npz")
    m, r, d, gamma, budget = _cfg(g)
    tr = [O.simulate_row(x, m, r, d, gamma, budget).sites for x in g["X"]]
    te = [O.simulate_row(x, m, r, d, gamma, budget).sites for x in g["X_test"]]
    assert np.array_equal(O.gram(te, tr, "test"), g["K_test"])
    amp = np.array([[O.overlap(a, b) for b in tr[:4]] for a in te[:4]])
    assert np.array_equal(amp, g["amp_test4"])


def test_oracle_gate_sequence_matches_reference():
    for name in ("config1_m8_d1.npz", "headline_m165_d1.npz", "config2_m50_d2.npz", "config3_m100_d4.npz"):
        g = golden(name)
        m, r, d, gamma, _ = _cfg(g)
        gates = O.feature_map_gates(g["X"][0], m, r, d, gamma)
        kinds = [("H", "RZ", "RXX", "SWAP").index(k) for k, _, _, _ in gates]
        assert np.array_equal(kinds, g["kinds"])
        assert np.array_equal([a for _, a, _, _ in gates], g["q0"])
        assert np.array_equal([b for _, _, b, _ in gates], g["q1"])
        ang = np.array([np.nan if a is None else a for *_, a in gates])
        assert np.array_equal(ang, g["angles0"], equal_nan=True)


def test_oracle_svd_rule_matches_reference():
    g = golden("svd_cases.npz")
    for mat, (rows, cols), budget, keep, sv, disc in zip(
        g["mats"], g["shapes"], g["budgets"], g["keeps"], g["svals"], g["discarded"]
    ):
        u, s, vh, dw = O.svd_truncated(np.asarray(mat).reshape(rows, cols), budget)
        assert s.size == keep
        assert np.array_equal(s, np.asarray(sv)[:keep])
        assert dw == disc


def test_oracle_kernel_fixture_and_dense():
    g = golden("kernel_fixture.npz")
    states = [O.simulate_row(x, 6, 1, 2, 0.5, 1e-24).sites for x in g["X"]]
    K = O.gram(states, states, "train")
    assert np.array_equal(K, g["K"])
    sv = g["statevectors"]
    dense = np.abs(sv.conj() @ sv.T) ** 2
    assert np.abs(K - dense).max() < 1e-10


def test_oracle_acceptance_c1_subset():
    cases = golden("acceptance_c1.json")
    for c in cases[:15]:
        X = np.array(c["X"])
        st = [O.simulate_row(x, c["m"], c["r"], c["d"], c["gamma"], 1e-24) for x in X]
        assert [s.bond_dims() for s in st] == c["chi"]
        assert np.array_equal(O.gram([s.sites for s in st], [s.sites for s in st], "train"), np.array(c["K"]))


def test_overlap_flops_formula():
    g = golden("headline_m165_d1.npz")
    chi = g["train_chi"]
    f = [O.overlap_flops(chi[i], chi[j]) for i in range(6) for j in range(i + 1, 6)]
    assert 8e4 < np.mean(f) < 1.5e5  # 1.108e5 mean at the headline shape
