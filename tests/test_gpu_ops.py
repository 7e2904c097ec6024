"""GPU drop-ins for the reference's state-level API (mps.py:123-247):
apply_one_qubit / apply_two_qubit / apply_gate / canonicalize / run_circuit
on GIVEN states, run as op programs continuing the state on the device
(mpskq_run_program, from_input=1), checked against the reference's own
results (tests/golden/ops_sequences.npz, made by make_golden.py --ops from
tests/golden/ops_cases.py).  Also: per-state chi-capacity escalation, the
per-phase timings, and the pinned host-K path of compute_gram /
run_distributed."""

import sys

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu
sys.path.insert(0, str(GOLDEN))


def test_state_ops_match_reference_sequences():
    import ops_cases

    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200 import ansatz, mps

    g = golden("ops_sequences.npz")
    for name, m, budget, steps in ops_cases.cases():
        st, log = ops_cases.run(mps, ansatz, m, budget, steps)
        assert st.bond_dims() == g[name + "_chi"].tolist(), name
        assert st.peak_chi == int(g[name + "_peak"]), name
        assert st.ortho_center == int(g[name + "_center"]), name
        assert [st.gate_count_1q, st.gate_count_2q] == g[name + "_counts"].tolist(), name
        assert log == g[name + "_memlog"].tolist(), name
        ref_disc = float(g[name + "_discard"])
        assert abs(st.accumulated_discard - ref_disc) <= 1e-9 * ref_disc + 1e-24, name
        # the state vector is gauge invariant: equal to rounding
        sv = P.to_statevector(st)
        assert np.abs(sv - g[name + "_sv"]).max() < 1e-10, name
        # phases recorded like MpsState.timings (mps.py:137, :159, :204)
        assert set(st.timings) <= {"canonicalize", "one_qubit", "two_qubit"}
        assert st.timings["two_qubit"] > 0 and st.timings["one_qubit"] > 0


def test_state_op_errors_match_reference():
    import paper_2411_09336_b200 as P

    st = P.init_state(4)
    with pytest.raises(ValueError, match="out of range"):
        P.apply_one_qubit(st, 4, np.eye(2))
    with pytest.raises(ValueError, match="2x2"):
        P.apply_one_qubit(st, 0, np.eye(3))
    with pytest.raises(ValueError, match="unitary"):
        P.apply_one_qubit(st, 0, np.array([[1.0, 1.0], [0.0, 1.0]]))
    with pytest.raises(ValueError, match="out of range"):
        P.apply_two_qubit(st, 3, np.eye(4))
    with pytest.raises(ValueError, match="absorb"):
        P.apply_two_qubit(st, 0, np.eye(4), absorb="up")
    with pytest.raises(ValueError, match="adjacent"):
        P.apply_gate(st, P.Gate("RXX", (0, 2), 0.3))
    with pytest.raises(ValueError, match="out of range"):
        P.canonicalize(st, 7)
    # the reference's bit-flip check (test_kernel.py:67-70)
    a, b = P.init_state(2), P.init_state(2)
    P.apply_one_qubit(b, 0, np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex))
    assert abs(P.inner_product(a, b)) < 1e-15
    assert abs(P.inner_product(b, b) - 1.0) < 1e-15


def test_canonicalize_from_unknown_center_gives_isometries():
    import paper_2411_09336_b200 as P

    g = golden("config1_m8_d1.npz")
    cfg = P.FeatureMapConfig(8, 2, 1, 0.5)
    st = P.simulate_dataset(g["X"][:1], cfg, budget=0.0)[0]
    sv0 = P.to_statevector(st)
    st.ortho_center = None  # full left + right sweeps (mps.py:129-131)
    P.canonicalize(st, 3)
    assert st.ortho_center == 3
    for s, t in enumerate(st.sites):
        if s < 3:
            mat = t.reshape(-1, t.shape[2])
            assert np.abs(mat.conj().T @ mat - np.eye(mat.shape[1])).max() < 1e-12
        elif s > 3:
            mat = t.reshape(t.shape[0], -1)
            assert np.abs(mat @ mat.conj().T - np.eye(mat.shape[0])).max() < 1e-12
    assert np.abs(P.to_statevector(st) - sv0).max() < 1e-12


def test_per_state_capacity_escalation():
    """All states start at capacity 4; only the ones that outgrow it move on
    (4 -> 8 -> 12) and the levels are gathered into one capacity-12 batch."""
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200 import mps

    g = golden("config2_m50_d2.npz")
    cfg = P.FeatureMapConfig(50, 2, 2, 0.1)
    mps._CAP_HINT.clear()
    b = P.simulate_dataset(g["X"], cfg, budget=1e-24)
    assert b.chi_cap == 12
    assert np.array_equal(b.bond_dims(), g["train_chi"])
    assert np.array_equal(b.peak.cpu().numpy(), g["train_peak"])
    K = P.compute_gram(b, b, "train").entries
    assert np.abs(K - g["K_train"]).max() < 1e-10
    from paper_2411_09336_b200.kernel import simulate_rows

    direct = simulate_rows(g["X"], cfg, 1e-24, chi_cap=12)
    Kd = P.compute_gram(direct, direct, "train").entries
    # capacities 8 and 12 run different lanes per state (32 lockstepped vs
    # 64), so the Jacobi's reduction order differs in the last bits
    assert np.abs(K - Kd).max() < 1e-12
    assert np.array_equal(direct.bond_dims(), b.bond_dims())


def test_run_distributed_single_gpu_is_the_native_path():
    import paper_2411_09336_b200 as P

    g = golden("headline_m165_d1.npz")
    cfg = P.FeatureMapConfig(165, 2, 1, 0.1)
    X = g["X"]
    rep = P.RunReport()
    gm = P.run_distributed(X, X, cfg, P.make_schedule(len(X), len(X), 2, "round_robin", "train"), report=rep)
    assert np.abs(gm.entries - g["K_train"]).max() < 1e-10
    assert np.all(np.diag(gm.entries) == 1.0) and np.array_equal(gm.entries, gm.entries.T)
    assert rep.n_simulations == len(X) and rep.n_inner_products == len(X) * (len(X) - 1) // 2
    assert rep.seconds["simulation"] > 0 and rep.seconds["inner_products"] > 0
    Xt = g["X_test"]
    gt = P.run_distributed(Xt, X, cfg, P.make_schedule(len(Xt), len(X), 1, "no_messaging", "test"))
    assert np.abs(gt.entries - g["K_test"]).max() < 1e-10
    # compute_gram's host path (pinned, banded) equals the device path bitwise
    tr = P.simulate_dataset(X, cfg)
    from paper_2411_09336_b200.mps import overlap_matrix

    Kh = P.compute_gram(tr, tr, "train").entries
    Kd = overlap_matrix(tr, tr, "train").cpu().numpy()
    assert np.array_equal(Kh, Kd)


def test_benchmark_reports_real_per_sample_times():
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200.benchmark import benchmark_rows

    cfg = P.FeatureMapConfig(12, 2, 2, 0.5)
    X = np.random.default_rng(5).uniform(0.0, 2.0, (6, 12))
    out = benchmark_rows(X, cfg)
    assert len(out["simulation_seconds"]) == 6 and len(out["inner_product_seconds"]) == 15
    assert all(t > 0 for t in out["simulation_seconds"] + out["inner_product_seconds"])
    assert len(set(out["simulation_seconds"])) > 1  # measured per sample, not a divided batch time
    with pytest.raises(ValueError, match="finite"):
        benchmark_rows(np.full((2, 12), np.nan), cfg)
    with pytest.raises(ValueError, match=r"\[0, 2\]"):
        benchmark_rows(np.full((2, 12), 3.0), cfg)


def test_run_distributed_row_errors_through_the_native_path():
    """Non-finite / out-of-range rows are caught by the device encoder of the
    one-GPU native call with the reference's messages (kernel.py:138-144,
    ansatz.py:121-124); non-finite wins when both occur."""
    import paper_2411_09336_b200 as P

    cfg = P.FeatureMapConfig(6, 1, 2, 0.5)
    X = np.random.default_rng(3).uniform(0.0, 2.0, (5, 6))
    sched = P.make_schedule(5, 5, 1, "round_robin", "train")
    bad = X.copy()
    bad[2, 3] = np.nan
    with pytest.raises(ValueError, match="finite"):
        P.run_distributed(bad, bad, cfg, sched)
    bad = X.copy()
    bad[4, 0] = 3.0
    with pytest.raises(ValueError, match=r"\[0, 2\]"):
        P.run_distributed(bad, bad, cfg, sched)
    bad[1, 1] = np.inf
    with pytest.raises(ValueError, match="finite"):
        P.run_distributed(bad, bad, cfg, sched)
    Xt = np.random.default_rng(4).uniform(0.0, 2.0, (2, 6))
    Xt[0, 0] = -0.5
    with pytest.raises(ValueError, match=r"\[0, 2\]"):
        P.run_distributed(Xt, X, cfg, P.make_schedule(2, 5, 1, "round_robin", "test"))
    # a good call after the failures still works (no sticky state)
    K = P.run_distributed(X, X, cfg, sched).entries
    assert np.all(np.diag(K) == 1.0)
