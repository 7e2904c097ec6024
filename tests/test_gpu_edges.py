"""Edge cases of the GPU path against the CPU oracle: tiny chains, single
states, ragged tile shapes, heavy truncation and the chi_max extension."""

import numpy as np
import pytest

from oracle import mps_oracle as O

pytestmark = pytest.mark.gpu


def _oracle_states(X, m, r, d, gamma, budget, chi_max=0):
    return [O.simulate_row(x, m, r, d, gamma, budget, chi_max) for x in X]


@pytest.mark.parametrize("m,d,n", [(2, 1, 1), (2, 1, 3), (3, 2, 5), (5, 1, 33), (7, 3, 41)])
def test_small_chains_and_ragged_counts(m, d, n):
    import paper_2411_09336_b200 as P

    rng = np.random.default_rng(m * 100 + n)
    X = rng.uniform(0.0, 2.0, (n, m))
    Xt = rng.uniform(0.0, 2.0, (max(1, n // 3), m))
    cfg = P.FeatureMapConfig(m, 2, d, 0.7)
    tr = P.simulate_dataset(X, cfg)
    te = P.simulate_dataset(Xt, cfg)
    ref = _oracle_states(X, m, 2, d, 0.7, 1e-24)
    reft = _oracle_states(Xt, m, 2, d, 0.7, 1e-24)
    assert tr.bond_dims().tolist() == [s.bond_dims() for s in ref]
    K = P.compute_gram(tr, tr, "train").entries
    Kt = P.compute_gram(te, tr, "test").entries
    assert K.shape == (n, n) and Kt.shape == (len(Xt), n)
    assert np.abs(K - O.gram([s.sites for s in ref], [s.sites for s in ref], "train")).max() < 1e-10
    assert np.abs(Kt - O.gram([s.sites for s in reft], [s.sites for s in ref], "test")).max() < 1e-10


def test_single_qubit_circuit():
    import paper_2411_09336_b200 as P

    circ = P.Circuit(1, [P.Gate("H", (0,)), P.Gate("RZ", (0,), 0.3), P.Gate("H", (0,))])
    st = P.simulate_circuit(circ, budget=0.0)
    ref = O.simulate_gates([("H", 0, -1, None), ("RZ", 0, -1, 0.3), ("H", 0, -1, None)], 1, 0.0)
    assert st.bond_dims() == [1, 1]
    assert np.allclose(st.sites[0], ref.sites[0], atol=1e-15)
    assert abs(P.inner_product(st, st) - 1) < 1e-15


@pytest.mark.parametrize("budget", [1e-6, 1e-3])
def test_heavy_truncation_matches_oracle(budget):
    """Coarse budgets truncate at almost every gate (renormalisation path)."""
    import paper_2411_09336_b200 as P

    X = np.random.default_rng(9).uniform(0.0, 2.0, (12, 20))
    cfg = P.FeatureMapConfig(20, 2, 3, 1.0)
    b = P.simulate_dataset(X, cfg, budget=budget)
    ref = _oracle_states(X, 20, 2, 3, 1.0, budget)
    assert b.bond_dims().tolist() == [s.bond_dims() for s in ref]
    assert np.allclose(b.discard.cpu().numpy(), [s.discard for s in ref], rtol=1e-8, atol=1e-20)
    K = P.compute_gram(b, b, "train").entries
    assert np.abs(K - O.gram([s.sites for s in ref], [s.sites for s in ref], "train")).max() < 1e-6


@pytest.mark.parametrize("chi_max", [2, 3, 5])
def test_chi_max_extension_matches_oracle_restatement(chi_max):
    """chi_max (BASELINE config 2) caps the kept rank; the oracle restates the
    same rule (oracle/mps_oracle.svd_truncated docstring)."""
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200.kernel import simulate_rows

    X = np.random.default_rng(2).uniform(0.0, 2.0, (10, 16))
    cfg = P.FeatureMapConfig(16, 2, 2, 0.5)
    b = simulate_rows(X, cfg, 1e-24, chi_max=chi_max)
    ref = _oracle_states(X, 16, 2, 2, 0.5, 1e-24, chi_max)
    assert b.bond_dims().max() <= chi_max
    assert b.bond_dims().tolist() == [s.bond_dims() for s in ref]
    K = P.compute_gram(b, b, "train").entries
    assert np.abs(K - O.gram([s.sites for s in ref], [s.sites for s in ref], "train")).max() < 1e-6


def test_mixed_capacity_batches_and_reference_states():
    """compute_gram between a GPU batch and uploaded host states of another
    capacity (the library re-packs to a common capacity)."""
    import paper_2411_09336_b200 as P

    X = np.random.default_rng(4).uniform(0.0, 2.0, (6, 10))
    cfg = P.FeatureMapConfig(10, 2, 2, 0.5)
    b = P.simulate_dataset(X, cfg)
    ref = _oracle_states(X[:3], 10, 2, 2, 0.5, 1e-24)
    host = [P.MpsState(s.sites) for s in ref]
    K = P.compute_gram(host, b, "test").entries
    Ko = O.gram([s.sites for s in ref], [s.sites for s in _oracle_states(X, 10, 2, 2, 0.5, 1e-24)], "test")
    assert np.abs(K - Ko).max() < 1e-12


def test_benchmark_payload_memory_series_matches_oracle():
    """benchmark_rows mirrors cmd_benchmark's payload (cli.py:240-294): the
    per-gate memory series and max chi equal the oracle's (= reference's)."""
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200.benchmark import benchmark_rows

    X = np.random.default_rng(12).uniform(0.0, 2.0, (5, 12))
    cfg = P.FeatureMapConfig(12, 2, 2, 0.5)
    out = benchmark_rows(X, cfg)
    ref = [O.simulate_gates(O.feature_map_gates(x, 12, 2, 2, 0.5), 12, 1e-24, record_memory=True) for x in X]
    assert out["memory_bytes_per_gate"] == [r.memory for r in ref]
    assert out["max_chi"] == [max(r.peak, max(r.bond_dims())) for r in ref]
    assert len(out["inner_product_seconds"]) == 10 and out["simulation_summary"]["median"] > 0
    with pytest.raises(ValueError):
        benchmark_rows(X[:1], cfg)


def test_long_chain_overlap_falls_back_to_a_shallower_ring():
    """m = 1000 qubits: the chi <= 4 overlap's 10-stage ring no longer fits
    shared memory next to the per-warp bond tables, so the 8-stage build runs;
    K against the oracle on a few states."""
    import paper_2411_09336_b200 as P

    m = 1000
    X = np.random.default_rng(21).uniform(0.0, 2.0, (40, m))
    cfg = P.FeatureMapConfig(m, 2, 1, 0.1)
    tr = P.simulate_dataset(X, cfg)
    assert tr.chi_cap == 4
    K = P.compute_gram(tr, tr, "train").entries
    ref = [O.simulate_row(X[i], m, 2, 1, 0.1, 1e-24) for i in (0, 1, 2)]
    assert [tr.bond_dims()[i].tolist() for i in (0, 1, 2)] == [r.bond_dims() for r in ref]
    Ko = O.gram([r.sites for r in ref], [r.sites for r in ref], "train")
    assert np.abs(K[:3, :3] - Ko).max() < 1e-10
    assert np.array_equal(K, K.T) and np.all(np.diag(K) == 1.0)
