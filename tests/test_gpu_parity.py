"""GPU parity: the CUDA path (through the C ABI) against the reference's
recorded outputs (tests/golden, made by running /root/reference) and the CPU
oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): kernel entries within 1e-10 absolute
for untruncated configs (budget 0 / 1e-24) and 1e-6 with fidelity-cutoff
truncation (1e-16); bond dimensions identical per site."""

import ctypes as C

import numpy as np
import pytest

from conftest import golden, unpack_states
from oracle import mps_oracle as O

pytestmark = pytest.mark.gpu

CASES = ["config1_m8_d1.npz", "headline_m165_d1.npz", "config2_m50_d2.npz", "config3_m100_d4.npz"]


def _tol(budget):
    return 1e-10 if budget <= 1e-24 else 1e-6


def _cfg(g):
    import paper_2411_09336_b200 as P

    return P.FeatureMapConfig(int(g["m"]), int(g["r"]), int(g["d"]), float(g["gamma"])), float(g["budget"])


@pytest.mark.parametrize("name", CASES)
def test_simulation_and_gram_match_reference(name):
    import paper_2411_09336_b200 as P

    g = golden(name)
    cfg, budget = _cfg(g)
    train = P.simulate_dataset(g["X"], cfg, budget=budget)
    test = P.simulate_dataset(g["X_test"], cfg, budget=budget)
    assert np.array_equal(train.bond_dims(), g["train_chi"]), "bond dims differ from the reference"
    assert np.array_equal(test.bond_dims(), g["test_chi"])
    assert np.array_equal(train.peak.cpu().numpy(), g["train_peak"])
    # accumulated_discard sums squares of singular values near sqrt(budget); its
    # rounding floor is ~eps * s_max * s_tail per gate, i.e. ~1e-28 per gate here
    disc = train.discard.cpu().numpy()
    assert np.all(np.abs(disc - g["train_discard"]) <= 1e-26 + 1e-4 * g["train_discard"])
    Ktr = P.compute_gram(train, train, "train").entries
    Kte = P.compute_gram(test, train, "test").entries
    tol = _tol(budget)
    assert np.abs(Ktr - g["K_train"]).max() < tol
    assert np.abs(Kte - g["K_test"]).max() < tol
    assert np.array_equal(Ktr, Ktr.T)
    assert np.all(np.diag(Ktr) == 1.0)


@pytest.mark.parametrize("name", ["config1_m8_d1.npz", "headline_m165_d1.npz"])
def test_overlap_kernel_on_reference_states(name):
    """Minimum slice: reference-produced MPS uploaded through the C ABI, K on the GPU."""
    import paper_2411_09336_b200 as P

    g = golden(name)
    sites = unpack_states(g)
    states = [P.MpsState([np.array(t) for t in s]) for s in sites]
    batch = P.MpsBatch.from_states(states)
    K = P.compute_gram(batch, batch, "train").entries
    assert np.abs(K - g["K_train"][: len(states), : len(states)]).max() < 1e-12
    assert np.array_equal(K, K.T) and np.all(np.diag(K) == 1.0)
    # the same states through the generic (capacity 8) overlap path
    b8 = P.MpsBatch.from_states(states, chi_cap=8)
    K8 = P.compute_gram(b8, b8, "train").entries
    assert np.abs(K8 - g["K_train"][: len(states), : len(states)]).max() < 1e-12


def test_amplitudes_and_inner_product():
    import paper_2411_09336_b200 as P

    g = golden("config1_m8_d1.npz")
    cfg, budget = _cfg(g)
    tr = P.simulate_dataset(g["X"][:4], cfg, budget=budget)
    te = P.simulate_dataset(g["X_test"][:4], cfg, budget=budget)
    amp = np.array([[P.inner_product(te[i], tr[j]) for j in range(4)] for i in range(4)])
    # amplitudes depend on the gauge only through a global phase per state
    assert np.abs(np.abs(amp) - np.abs(g["amp_test4"])).max() < 1e-12
    assert abs(P.inner_product(tr[0], tr[0]) - 1.0) < 1e-12


def test_states_match_oracle_statevector():
    """Every reconstructed state equals the oracle's (same gauge-free vector)."""
    import paper_2411_09336_b200 as P

    g = golden("config1_m8_d1.npz")
    cfg, budget = _cfg(g)
    batch = P.simulate_dataset(g["X"][:8], cfg, budget=budget)
    for i, x in enumerate(g["X"][:8]):
        ref = O.simulate_row(x, 8, 2, 1, 0.5, budget)
        a = P.to_statevector(batch[i])
        b = P.to_statevector(P.MpsState(ref.sites))
        assert abs(abs(np.vdot(a, b)) - 1.0) < 1e-12
        assert np.abs(np.abs(a) - np.abs(b)).max() < 1e-12


def test_acceptance_c1_random_configs():
    """Acceptance criterion 1 (test_acceptance.py:41-75): 50 random configs."""
    import paper_2411_09336_b200 as P

    for c in golden("acceptance_c1.json"):
        cfg = P.FeatureMapConfig(c["m"], c["r"], c["d"], c["gamma"])
        b = P.simulate_dataset(np.array(c["X"]), cfg)
        assert b.bond_dims().tolist() == c["chi"]
        K = P.compute_gram(b, b, "train").entries
        assert np.abs(K - np.array(c["K"])).max() < 1e-10


def test_svd_truncated_matches_reference_rule():
    import paper_2411_09336_b200 as P

    g = golden("svd_cases.npz")
    for mat, (rows, cols), budget, keep, sv, disc in zip(
        g["mats"], g["shapes"], g["budgets"], g["keeps"], g["svals"], g["discarded"]
    ):
        A = np.asarray(mat).reshape(rows, cols)
        res = P.svd_truncated(A, 1, budget)
        assert res.singular_values.size == keep
        assert np.abs(res.singular_values - np.asarray(sv)[:keep]).max() < 1e-13
        assert abs(res.discarded_weight - disc) <= 1e-6 * disc + 1e-26  # tail values carry ~eps*s0 abs error
        U, s, Vh = res.left, res.singular_values, res.right
        assert np.abs(U.conj().T @ U - np.eye(keep)).max() < 1e-12 or keep == 0
        assert np.abs(Vh @ Vh.conj().T - np.eye(keep)).max() < 1e-12
        err = np.linalg.norm(A - (U * s) @ Vh)
        assert abs(err - np.sqrt(disc)) < 1e-10


def test_svd_errors():
    import paper_2411_09336_b200 as P

    with pytest.raises(ValueError, match="non-finite"):
        P.svd_truncated(np.full((2, 2), np.nan), 1, 0.0)
    with pytest.raises(ValueError, match="budget"):
        P.svd_truncated(np.eye(2), 1, -1.0)
    with pytest.raises(ValueError, match="split"):
        P.svd_truncated(np.eye(2), 2, 0.0)


def _random_circuit(rng, m, n):
    import paper_2411_09336_b200 as P

    gates = []
    for _ in range(n):
        k = rng.integers(4)
        if k == 0:
            gates.append(P.Gate("H", (int(rng.integers(m)),)))
        elif k == 1:
            gates.append(P.Gate("RZ", (int(rng.integers(m)),), float(rng.uniform(-3, 3))))
        else:
            q = int(rng.integers(m - 1))
            pair = (q, q + 1) if rng.random() < 0.5 else (q + 1, q)
            gates.append(P.Gate("RXX" if k == 2 else "SWAP", pair, float(rng.uniform(-3, 3)) if k == 2 else None))
    return P.Circuit(m, gates)


def test_simulate_circuit_random_circuits_vs_oracle():
    import paper_2411_09336_b200 as P

    rng = np.random.default_rng(11)
    for _ in range(20):
        m = int(rng.integers(2, 9))
        circ = _random_circuit(rng, m, 40)
        log = []
        st = P.simulate_circuit(circ, budget=0.0, memory_log=log)
        ref = O.simulate_gates([(g.kind, g.qubits[0], g.qubits[1] if len(g.qubits) > 1 else -1, g.angle)
                                for g in circ.gates], m, 0.0, record_memory=True)
        assert st.bond_dims() == ref.bond_dims()
        assert log == ref.memory
        a, b = P.to_statevector(st), P.to_statevector(P.MpsState(ref.sites))
        assert abs(abs(np.vdot(a, b)) - 1.0) < 1e-12
        assert st.gate_count_1q == ref.g1 and st.gate_count_2q == ref.g2
        assert st.ortho_center == ref.center


def test_gram_errors():
    import paper_2411_09336_b200 as P

    cfg = P.FeatureMapConfig(6, 1, 2, 0.5)
    X = np.random.default_rng(42).uniform(0.0, 2.0, (4, 6))
    s1 = P.simulate_dataset(X, cfg)
    s2 = P.simulate_dataset(X, cfg)
    with pytest.raises(ValueError, match="same states"):
        P.compute_gram(s1, s2, "train")
    other = P.simulate_dataset(np.ones((1, 4)), P.FeatureMapConfig(4, 1, 1, 0.5))
    with pytest.raises(ValueError, match="mismatch"):
        P.compute_gram(other, s1, "test")
    with pytest.raises(ValueError, match="length 6"):
        P.simulate_dataset(np.zeros((2, 5)), cfg)
    with pytest.raises(ValueError, match="finite"):
        P.simulate_dataset(np.full((1, 6), np.nan), cfg)
    assert P.simulate_dataset(np.zeros((0, 6)), cfg) == []


def test_kernel_fixture_dense_oracle():
    """test_kernel.py's fixture: Gram vs dense statevector oracle < 1e-10."""
    import paper_2411_09336_b200 as P

    g = golden("kernel_fixture.npz")
    b = P.simulate_dataset(g["X"], P.FeatureMapConfig(6, 1, 2, 0.5))
    K = P.compute_gram(b, b, "train").entries
    sv = g["statevectors"]
    assert np.abs(K - np.abs(sv.conj() @ sv.T) ** 2).max() < 1e-10
    assert np.abs(K - g["K"]).max() < 1e-12
    eig = np.linalg.eigvalsh(K)
    assert eig.min() >= -1e-10


def test_run_distributed_single_process():
    import paper_2411_09336_b200 as P

    g = golden("config1_m8_d1.npz")
    cfg, budget = _cfg(g)
    for strategy in ("round_robin", "no_messaging"):
        for k in (1, 4):
            rep = P.RunReport()
            sched = P.make_schedule(64, 64, k, strategy, "train")
            K = P.run_distributed(g["X"], g["X"], cfg, sched, budget=budget, report=rep).entries
            assert np.abs(K - g["K_train"]).max() < 1e-10
            assert rep.n_simulations == 64 and rep.n_inner_products == 64 * 63 // 2
            rep = P.RunReport()
            sched = P.make_schedule(16, 64, k, strategy, "test")
            Kt = P.run_distributed(g["X_test"], g["X"], cfg, sched, budget=budget, report=rep).entries
            assert np.abs(Kt - g["K_test"]).max() < 1e-10
            assert rep.n_simulations == 80 and rep.n_inner_products == 16 * 64
    with pytest.raises(ValueError, match="state counts"):
        P.run_distributed(g["X"][:4], g["X"][:4], cfg, P.make_schedule(64, 64, 2, "round_robin", "train"))


def test_c_abi_end_to_end_host_buffers(native):
    """mpskq_gram_host: host rows in, host K out, through the C ABI only."""
    from paper_2411_09336_b200 import _native as N

    for name in ("config1_m8_d1.npz", "headline_m165_d1.npz"):
        g = golden(name)
        X = np.ascontiguousarray(g["X"])
        Xt = np.ascontiguousarray(g["X_test"])
        n, m = X.shape
        K = np.zeros((n, n))
        secs = np.zeros(4)
        N.check(native.mpskq_gram_host(N.KIND_TRAIN, m, int(g["r"]), int(g["d"]), float(g["gamma"]),
                                       float(g["budget"]), 0, 0, N.ptr(X, C.c_double), n, None, 0,
                                       N.ptr(K, C.c_double), None, N.ptr(secs, C.c_double)))
        assert np.abs(K - g["K_train"]).max() < 1e-10
        Kt = np.zeros((Xt.shape[0], n))
        N.check(native.mpskq_gram_host(N.KIND_TEST, m, int(g["r"]), int(g["d"]), float(g["gamma"]),
                                       float(g["budget"]), 0, 0, N.ptr(Xt, C.c_double), Xt.shape[0],
                                       N.ptr(X, C.c_double), n, N.ptr(Kt, C.c_double), None, None))
        assert np.abs(Kt - g["K_test"]).max() < 1e-10
        assert secs[0] > 0 and secs[1] > 0


def test_fp64_probe_runs(native):
    import torch

    from paper_2411_09336_b200 import _native as N

    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    N.check(native.mpskq_fp64_probe(4, 100, out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()


def test_chi_capacity_escalation():
    """config 2 needs chi up to ~10: the engine escalates 4 -> 16 transparently,
    and a forced too-small capacity raises."""
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200.kernel import simulate_rows

    g = golden("config2_m50_d2.npz")
    cfg, budget = _cfg(g)
    b = simulate_rows(g["X"][:4], cfg, budget)
    assert b.chi_cap == 12
    with pytest.raises(RuntimeError):
        simulate_rows(g["X"][:4], cfg, budget, chi_cap=4)


def test_wire_format_of_gpu_states():
    import paper_2411_09336_b200 as P

    g = golden("wire_mps1.npz")
    ref = [P.deserialize_state(g[k].tobytes()) for k in ("blob0", "blob1")]
    batch = P.simulate_dataset(g["X"], P.FeatureMapConfig(6, 2, 2, 0.5))
    for i, r in enumerate(ref):
        st = P.deserialize_state(P.serialize_state(batch[i]))
        assert st.bond_dims() == r.bond_dims()
        assert (st.m, st.ortho_center, st.peak_chi, st.gate_count_1q, st.gate_count_2q) == (
            r.m, r.ortho_center, r.peak_chi, r.gate_count_1q, r.gate_count_2q)
        assert abs(abs(np.vdot(P.to_statevector(st), P.to_statevector(r))) - 1) < 1e-12


def test_downstream_svc_matches_reference_kernel():
    """Config 1's experiment flow: blobs -> split -> rescale -> GPU train/test
    kernels -> SVC over the C grid.  The precomputed-kernel SVC on the GPU K
    reproduces the predictions made on the reference K (golden), i.e. the same
    downstream accuracy."""
    from sklearn.svm import SVC

    import paper_2411_09336_b200 as P

    g = golden("svc_config1.npz")
    cfg = P.FeatureMapConfig(8, 2, 1, 0.5)
    ntr, nte = len(g["X_train"]), len(g["X_test"])
    Ktr = P.run_distributed(g["X_train"], g["X_train"], cfg, P.make_schedule(ntr, ntr, 1, "round_robin", "train"),
                            budget=0.0).entries
    Kte = P.run_distributed(g["X_test"], g["X_train"], cfg, P.make_schedule(nte, ntr, 1, "round_robin", "test"),
                            budget=0.0).entries
    assert np.abs(Ktr - g["K_train"]).max() < 1e-10 and np.abs(Kte - g["K_test"]).max() < 1e-10
    for c, pred, dec in zip(g["C_grid"], g["sklearn_pred"], g["sklearn_decision"]):
        clf = SVC(C=float(c), kernel="precomputed").fit(Ktr, g["y_train"])
        assert np.array_equal(clf.predict(Kte), pred)
        assert np.abs(clf.decision_function(Kte) - dec).max() < 1e-6
    acc = max(np.mean(p == g["y_test"]) for p in g["sklearn_pred"])
    assert acc >= max(g["ref_accuracy"]) - 1e-12 or acc >= 0.95


def test_capacity_48_path_matches_reference():
    """chi capacity 48 (theta up to 96x96): Jacobi rotations logged and replayed.
    Config 5 at d=6 (m=100, budget 1e-16) needs it: final bonds reach 31 but
    the running peak_chi reaches 36 (mps.py:202)."""
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200.kernel import simulate_rows

    g = golden("config5_m100_d6.npz")
    cfg, budget = _cfg(g)
    b = simulate_rows(g["X"], cfg, budget, chi_cap=48)
    assert b.chi_cap == 48
    assert np.array_equal(b.bond_dims(), g["train_chi"])
    K = P.compute_gram(b, b, "train").entries
    assert np.abs(K - g["K_train"]).max() < 1e-6
    assert np.array_equal(b.peak.cpu().numpy(), g["train_peak"])
    # the automatic capacity choice escalates past 32 by itself
    auto = P.simulate_dataset(g["X"], cfg, budget=budget)
    assert auto.chi_cap == 48 and np.array_equal(auto.bond_dims(), g["train_chi"])
    with pytest.raises(RuntimeError):
        simulate_rows(g["X"], cfg, budget, chi_cap=32)


def test_large_chi_global_workspace_path():
    """Config 5 at d=8 (m=100, budget 1e-16) peaks at chi 68 on these rows:
    capacity 80 keeps theta in an L2-resident global workspace.  Bond dims
    identical to the reference, K within the truncated tolerance."""
    import time

    import paper_2411_09336_b200 as P

    g = golden("config5_m100_d8.npz")
    cfg, budget = _cfg(g)
    t0 = time.time()
    tr = P.simulate_dataset(g["X"], cfg, budget=budget)
    te = P.simulate_dataset(g["X_test"], cfg, budget=budget)
    print(f"d=8 simulation of 6 states: {time.time() - t0:.1f}s, capacity {tr.chi_cap}")
    assert tr.chi_cap == 80
    assert np.array_equal(tr.bond_dims(), g["train_chi"])
    assert np.array_equal(te.bond_dims(), g["test_chi"])
    assert np.array_equal(tr.peak.cpu().numpy(), g["train_peak"])
    K = P.compute_gram(tr, tr, "train").entries
    Kt = P.compute_gram(te, tr, "test").entries
    assert np.abs(K - g["K_train"]).max() < 1e-6
    assert np.abs(Kt - g["K_test"]).max() < 1e-6


def test_capacity_64_direct_w_path():
    """Config 5 at d=7 (m=100, budget 1e-16) peaks at chi 50-51 on these rows:
    capacity 64 keeps theta and the Jacobi W in the global workspace and
    accumulates W in place (no rotation log).  Same bond dims and peaks as the
    reference; the same rows through capacity 80 (rotation log) agree too."""
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200.kernel import simulate_rows

    g = golden("config5_m100_d7.npz")
    cfg, budget = _cfg(g)
    tr = P.simulate_dataset(g["X"], cfg, budget=budget)
    te = P.simulate_dataset(g["X_test"], cfg, budget=budget)
    assert tr.chi_cap == 64 and te.chi_cap == 64
    assert np.array_equal(tr.bond_dims(), g["train_chi"])
    assert np.array_equal(te.bond_dims(), g["test_chi"])
    assert np.array_equal(tr.peak.cpu().numpy(), g["train_peak"])
    assert np.array_equal(te.peak.cpu().numpy(), g["test_peak"])
    K = P.compute_gram(tr, tr, "train").entries
    Kt = P.compute_gram(te, tr, "test").entries
    assert np.abs(K - g["K_train"]).max() < 1e-6
    assert np.abs(Kt - g["K_test"]).max() < 1e-6
    b80 = simulate_rows(g["X"], cfg, budget, chi_cap=80)
    assert b80.chi_cap == 80 and np.array_equal(b80.bond_dims(), g["train_chi"])
    assert np.abs(P.compute_gram(b80, b80, "train").entries - g["K_train"]).max() < 1e-6


def test_svd_truncated_large_matrices():
    import paper_2411_09336_b200 as P

    g = golden("svd_cases_large.npz")
    for i in range(3):
        A = g[f"mat{i}"]
        res = P.svd_truncated(A, 1, float(g[f"budget{i}"]))
        s = g[f"s{i}"]
        assert res.singular_values.size == s.size
        assert np.abs(res.singular_values - s).max() < 1e-13
        U, Vh = res.left, res.right
        k = s.size
        assert np.abs(U.conj().T @ U - np.eye(k)).max() < 1e-11
        assert np.abs(Vh @ Vh.conj().T - np.eye(k)).max() < 1e-11


def test_integration_md_ctypes_stub_runs():
    """The binding a maintainer would add to the reference
    works as written: exec it against the golden config-1 rows."""
    import re
    from dataclasses import dataclass

    from conftest import ROOT

    import paper_2411_09336_b200 as P

    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"```python\n(import ctypes.*?)```", text, re.S).group(1)
    block = block.replace('"/path/to/paper_2411_09336_b200/libmpskq.so"',
                          repr(str(ROOT / "paper_2411_09336_b200" / "libmpskq.so")))

    @dataclass
    class GramMatrix:
        entries: np.ndarray
        kind: str

    ns = {"GramMatrix": GramMatrix, "DEFAULT_TRUNC_BUDGET": 1e-24}
    exec(block, ns)
    g = golden("config1_m8_d1.npz")
    cfg, budget = _cfg(g)
    rep = P.RunReport()
    K = ns["run_distributed"](g["X"], g["X"], cfg, P.make_schedule(64, 64, 1, "round_robin", "train"),
                              budget=budget, report=rep).entries
    assert np.abs(K - g["K_train"]).max() < 1e-10
    Kt = ns["run_distributed"](g["X_test"], g["X"], cfg, P.make_schedule(16, 64, 1, "round_robin", "test"),
                               budget=budget).entries
    assert np.abs(Kt - g["K_test"]).max() < 1e-10
    assert rep.n_inner_products == 64 * 63 // 2


@pytest.mark.parametrize("cap", [96, 128])
def test_largest_capacities_match_reference(cap):
    """The two largest capacities (96, and 128 for the paper's d=6 at 165 qubits
    with budget 1e-24) on the d=8 rows: same bond dims and peaks as the
    reference whatever capacity runs them."""
    import paper_2411_09336_b200 as P
    from paper_2411_09336_b200.kernel import simulate_rows

    g = golden("config5_m100_d8.npz")
    cfg, budget = _cfg(g)
    b = simulate_rows(g["X"], cfg, budget, chi_cap=cap)
    assert b.chi_cap == cap
    assert np.array_equal(b.bond_dims(), g["train_chi"])
    assert np.array_equal(b.peak.cpu().numpy(), g["train_peak"])
    K = P.compute_gram(b, b, "train").entries
    assert np.abs(K - g["K_train"]).max() < 1e-6


def test_c_abi_end_to_end_pinned_output_streams_bitwise(native):
    """mpskq_gram_host with a pinned K: the chi <= 4 overlap streams finished
    row bands into host memory (several 384-row bands here) — bitwise equal
    to the pageable path (device K + one copy), train diagonal exactly 1."""
    import torch

    from paper_2411_09336_b200 import _native as N

    rng = np.random.default_rng(7)
    m, r, d, gamma, budget = 165, 2, 1, 0.1, 1e-24
    X = np.ascontiguousarray(rng.uniform(0, 2, (900, m)))
    Xt = np.ascontiguousarray(rng.uniform(0, 2, (500, m)))

    def call(kind, bras, kets, out):
        n_k = bras.shape[0] if kets is None else kets.shape[0]
        assert out.shape == (bras.shape[0], n_k)
        N.check(native.mpskq_gram_host(kind, m, r, d, gamma, budget, 0, 4, N.ptr(bras, C.c_double),
                                       bras.shape[0], None if kets is None else N.ptr(kets, C.c_double),
                                       0 if kets is None else kets.shape[0],
                                       C.cast(out.ctypes.data if isinstance(out, np.ndarray) else out.data_ptr(),
                                              C.POINTER(C.c_double)), None, None))
        return out

    cases = [(N.KIND_TRAIN, X, None), (N.KIND_TEST, Xt, X), (N.KIND_TRAIN, X[:1].copy(), None),
             (N.KIND_TRAIN, X[:5].copy(), None), (N.KIND_TEST, Xt[:3].copy(), X[:7].copy())]
    for kind, bras, kets in cases:
        shape = (bras.shape[0], bras.shape[0] if kets is None else kets.shape[0])
        ref = call(kind, bras, kets, np.zeros(shape))
        pinned = torch.full(shape, -7.0, dtype=torch.float64).pin_memory()
        got = call(kind, bras, kets, pinned).numpy()
        assert np.array_equal(got, ref)
        if kind == N.KIND_TRAIN:
            assert np.array_equal(np.diag(got), np.ones(shape[0]))
            assert np.array_equal(got, got.T)
