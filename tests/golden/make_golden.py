"""Generate the golden fixtures of the parity suite from the REAL reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records its outputs for seeded inputs into tests/golden/*.npz.  The GPU box
never reads /root/reference: the tests only load these committed files.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

from mpskernel import ansatz, kernel, mps, tensor  # noqa: E402


def pack_states(states):
    """Flatten a list of MpsState into arrays (bond dims, offsets, entries)."""
    m = states[0].m
    chi = np.array([s.bond_dims() for s in states], dtype=np.int32)
    data, offs = [], []
    off = 0
    for s in states:
        row = []
        for t in s.sites:
            row.append(off)
            data.append(t.reshape(-1))
            off += t.size
        offs.append(row)
    return dict(
        chi=chi,
        site_off=np.array(offs, dtype=np.int64).reshape(len(states), m),
        entries=np.concatenate(data).astype(np.complex128),
        discard=np.array([s.accumulated_discard for s in states]),
        peak=np.array([s.peak_chi for s in states], dtype=np.int32),
        g1=np.array([s.gate_count_1q for s in states], dtype=np.int64),
        g2=np.array([s.gate_count_2q for s in states], dtype=np.int64),
    )


def gram_case(name, m, r, d, gamma, budget, n_train, n_test, seed, keep_states=False):
    t0 = time.time()
    cfg = ansatz.FeatureMapConfig(m, r, d, gamma)
    rng = np.random.default_rng(seed)
    X = rng.uniform(0.0, 2.0, (n_train, m))
    Xt = rng.uniform(0.0, 2.0, (n_test, m))
    train = kernel.simulate_dataset(X, cfg, budget=budget)
    test = kernel.simulate_dataset(Xt, cfg, budget=budget)
    Ktr = kernel.compute_gram(train, train, "train").entries
    Kte = kernel.compute_gram(test, train, "test").entries
    amp = np.array([[mps.inner_product(a, b) for b in train[:4]] for a in test[:4]])
    circ = ansatz.encode_circuit(X[0], cfg)
    out = dict(
        m=m, r=r, d=d, gamma=gamma, budget=budget, X=X, X_test=Xt, K_train=Ktr, K_test=Kte,
        amp_test4=amp,
        kinds=np.array([ansatz.GATE_KINDS.index(g.kind) for g in circ.gates], dtype=np.int32),
        q0=np.array([g.qubits[0] for g in circ.gates], dtype=np.int32),
        q1=np.array([g.qubits[1] if len(g.qubits) > 1 else -1 for g in circ.gates], dtype=np.int32),
        angles0=np.array([np.nan if g.angle is None else g.angle for g in circ.gates]),
    )
    for key, val in pack_states(train).items():
        if key in ("entries", "site_off") and not keep_states:
            continue
        out["train_" + key] = val
    for key, val in pack_states(test).items():
        if key in ("entries", "site_off"):
            continue
        out["test_" + key] = val
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: {time.time() - t0:.1f}s  max chi {out['train_chi'].max()}")


def svd_cases():
    """svd_truncated on matrices with prescribed spectra (tensor.py:87-123)."""
    rng = np.random.default_rng(7)
    mats, budgets, keeps, svals, discs, shapes = [], [], [], [], [], []

    def rand_unitary(n):
        q, _ = np.linalg.qr(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)))
        return q

    specs = [
        (4, 4, [1.0, 0.5, 0.25, 0.125], 0.0),
        (4, 4, [1.0, 0.5, 1e-9, 0.0], 0.0),
        (4, 4, [1.0, 0.5, 1e-9, 1e-18], 1e-30),
        (4, 4, [1.0, 1e-13, 1e-13, 1e-13], 1e-24),
        (8, 8, [1.0, 0.3, 0.1, 1e-5, 1e-8, 1e-11, 1e-13, 1e-16], 1e-24),
        (8, 6, [1.0, 0.3, 0.1, 1e-5, 1e-8, 1e-11], 1e-16),
        (6, 8, [1.0, 0.3, 0.1, 1e-5, 1e-8, 1e-11], 1e-20),
        (8, 8, [1.0] * 8, 0.5),
        (8, 8, [1.0] + [1e-16] * 7, 0.0),
        (16, 16, list(np.geomspace(1.0, 1e-15, 16)), 1e-24),
        (32, 32, list(np.geomspace(1.0, 1e-14, 32)), 1e-16),
        (16, 12, list(np.geomspace(1.0, 1e-10, 12)), 1e-18),
    ]
    for rows, cols, sv, budget in specs:
        k = min(rows, cols)
        u = rand_unitary(rows)[:, :k]
        v = rand_unitary(cols)[:k, :]
        mat = (u * np.array(sv)) @ v
        res = tensor.svd_truncated(mat.reshape(rows, cols), 1, budget)
        mats.append(mat.reshape(-1))
        budgets.append(budget)
        keeps.append(res.singular_values.size)
        s = np.zeros(k)
        s[: res.singular_values.size] = res.singular_values
        svals.append(s)
        discs.append(res.discarded_weight)
        shapes.append((rows, cols))
    np.savez_compressed(
        OUT / "svd_cases.npz",
        mats=np.array(mats, dtype=object),
        shapes=np.array(shapes, dtype=np.int32),
        budgets=np.array(budgets),
        keeps=np.array(keeps, dtype=np.int32),
        svals=np.array(svals, dtype=object),
        discarded=np.array(discs),
        allow_pickle=True,
    )
    print("svd_cases:", len(specs))


def schedule_cases():
    """make_schedule outputs for API parity (kernel.py:316-333)."""
    rows = []
    for strategy in ("round_robin", "no_messaging"):
        for kind, nb, nk in [("train", 5, 5), ("train", 16, 16), ("test", 4, 16), ("test", 3, 10)]:
            for k in (1, 2, 3, 4, 6):
                s = kernel.make_schedule(nb, nk, k, strategy, kind)
                tiles = [
                    (si, t.worker, t.row_start, t.row_stop, t.col_start, t.col_stop)
                    for si, st in enumerate(s.steps)
                    for t in st.tiles
                ]
                transfers = [
                    (si, t.src, t.dst, t.which, t.start, t.stop)
                    for si, st in enumerate(s.steps)
                    for t in st.transfers
                ]
                rows.append(
                    dict(strategy=strategy, kind=kind, nb=nb, nk=nk, k=k, kk=s.k,
                         initial={str(w): v for w, v in s.initial_states.items()},
                         tiles=tiles, transfers=transfers)
                )
    import json

    (OUT / "schedules.json").write_text(json.dumps(rows))
    print("schedules:", len(rows))


def kernel_fixture():
    """The reference's own test fixture: test_kernel.py:23-34 (m=6, r=1, d=2, gamma=0.5)."""
    cfg = ansatz.FeatureMapConfig(6, 1, 2, 0.5)
    X = np.random.default_rng(42).uniform(0.0, 2.0, (8, 6))
    states = kernel.simulate_dataset(X, cfg)
    K = kernel.compute_gram(states, states, "train").entries
    sv = [mps.to_statevector(s) for s in states]
    np.savez_compressed(OUT / "kernel_fixture.npz", X=X, K=K, chi=np.array([s.bond_dims() for s in states]),
                        statevectors=np.array(sv))
    print("kernel_fixture")


def acceptance_c1():
    """Acceptance criterion 1's random small configs (test_acceptance.py:41-75), seed 20240901."""
    rng = np.random.default_rng(20240901)
    cases = []
    for _ in range(50):
        m = int(rng.integers(2, 11))
        d = int(rng.integers(1, min(4, m - 1) + 1))
        r = int(rng.integers(1, 4))
        gamma = float(rng.choice([0.1, 0.5, 1.0]))
        X = rng.uniform(0.0, 2.0, (3, m))
        cfg = ansatz.FeatureMapConfig(m, r, d, gamma)
        states = kernel.simulate_dataset(X, cfg)
        K = kernel.compute_gram(states, states, "train").entries
        cases.append(dict(m=m, r=r, d=d, gamma=gamma, X=X.tolist(), K=K.tolist(),
                          chi=[s.bond_dims() for s in states],
                          discard=[s.accumulated_discard for s in states]))
    import json

    (OUT / "acceptance_c1.json").write_text(json.dumps(cases))
    print("acceptance_c1:", len(cases))


if __name__ == "__main__" and len(sys.argv) == 1:
    OUT.mkdir(parents=True, exist_ok=True)
    svd_cases()
    schedule_cases()
    kernel_fixture()
    acceptance_c1()
    # config 1: m=8, d=1 (BASELINE "r=1" = interaction distance), 2 layers, untruncated
    gram_case("config1_m8_d1", 8, 2, 1, 0.5, 0.0, 64, 16, seed=0, keep_states=True)
    # headline shape (config 4), subset of rows: m=165, d=1, 2 layers, gamma 0.1, budget 1e-24
    gram_case("headline_m165_d1", 165, 2, 1, 0.1, 1e-24, 24, 8, seed=0, keep_states=True)
    # config 2 shape: m=50, d=2, budget 1e-24
    gram_case("config2_m50_d2", 50, 2, 2, 0.1, 1e-24, 24, 8, seed=0)
    # config 3 shape: m=100, d=4, fidelity cutoff 1e-16
    gram_case("config3_m100_d4", 100, 2, 4, 0.1, 1e-16, 10, 4, seed=0)


def svc_experiment():
    """Config 1's experiment flow (cli.cmd_experiment, cli.py:152-214): blobs ->
    balanced split -> rescale -> train/test kernels -> SMO SVM over the C grid.
    Records the reference's K and downstream metrics, plus sklearn's
    precomputed-kernel SVC on the reference K (the GPU test reruns sklearn on
    the GPU K and must reproduce these)."""
    from mpskernel import cli, learn
    from sklearn.svm import SVC

    ds = cli.generate_blobs(cli.SyntheticSpec(n_per_class=40), m=8, seed=0)
    train, test = learn.split(ds, 0.8, seed=0)
    X_tr, X_te, _ = learn.rescale(train.features, test.features)
    cfg = ansatz.FeatureMapConfig(8, 2, 1, 0.5)
    gtr = kernel.run_distributed(X_tr, X_tr, cfg, kernel.make_schedule(len(X_tr), len(X_tr), 1, "round_robin", "train"), budget=0.0)
    gte = kernel.run_distributed(X_te, X_tr, cfg, kernel.make_schedule(len(X_te), len(X_tr), 1, "round_robin", "test"), budget=0.0)
    grid = np.geomspace(0.01, 4.0, 8)
    ref_auc, ref_acc, sk_pred, sk_dec = [], [], [], []
    for C in grid:
        model = learn.svm_train(gtr, train.labels, float(C))
        met = learn.evaluate(learn.decision_scores(model, gte), test.labels)
        ref_auc.append(met.auc)
        ref_acc.append(met.accuracy)
        clf = SVC(C=float(C), kernel="precomputed").fit(gtr.entries, train.labels)
        sk_pred.append(clf.predict(gte.entries))
        sk_dec.append(clf.decision_function(gte.entries))
    np.savez_compressed(
        OUT / "svc_config1.npz", X_train=X_tr, X_test=X_te, y_train=train.labels, y_test=test.labels,
        K_train=gtr.entries, K_test=gte.entries, C_grid=grid, ref_auc=np.array(ref_auc),
        ref_accuracy=np.array(ref_acc), sklearn_pred=np.array(sk_pred), sklearn_decision=np.array(sk_dec),
    )
    print("svc_config1: best ref AUC", max(ref_auc))


def wire_format():
    """serialize_state bytes of two reference states (mps.py:294-314)."""
    cfg = ansatz.FeatureMapConfig(6, 2, 2, 0.5)
    X = np.random.default_rng(8).uniform(0.0, 2.0, (2, 6))
    states = kernel.simulate_dataset(X, cfg)
    blobs = [np.frombuffer(mps.serialize_state(s), dtype=np.uint8) for s in states]
    np.savez_compressed(OUT / "wire_mps1.npz", X=X, blob0=blobs[0], blob1=blobs[1])
    print("wire_mps1")


if __name__ == "__main__" and "--extra" in sys.argv:
    svc_experiment()
    wire_format()


if __name__ == "__main__" and "--large-chi" in sys.argv:
    # config 5 (interaction-distance sweep at m=100, budget 1e-16): d=6 and d=8
    # need chi > 32, i.e. the capacity-48 path
    gram_case("config5_m100_d6", 100, 2, 6, 0.1, 1e-16, 4, 2, seed=0)
    gram_case("config5_m100_d8", 100, 2, 8, 0.1, 1e-16, 4, 2, seed=0)


if __name__ == "__main__" and "--d7" in sys.argv:
    # config 5 at d=7: peak chi 49-64, i.e. the capacity-64 path (theta and W
    # in the global workspace, no rotation log)
    gram_case("config5_m100_d7", 100, 2, 7, 0.1, 1e-16, 4, 2, seed=0)


def svd_cases_large():
    """svd_truncated on 65..96-sized matrices (the capacity-48 device path)."""
    rng = np.random.default_rng(77)
    out = {}
    for idx, (rows, cols, budget) in enumerate([(80, 80, 1e-16), (96, 90, 1e-24), (70, 96, 1e-20)]):
        k = min(rows, cols)
        q1, _ = np.linalg.qr(rng.normal(size=(rows, rows)) + 1j * rng.normal(size=(rows, rows)))
        q2, _ = np.linalg.qr(rng.normal(size=(cols, cols)) + 1j * rng.normal(size=(cols, cols)))
        sv = np.geomspace(1.0, 1e-14, k)
        mat = (q1[:, :k] * sv) @ q2[:k, :]
        res = tensor.svd_truncated(mat, 1, budget)
        out[f"mat{idx}"] = mat
        out[f"budget{idx}"] = budget
        out[f"s{idx}"] = res.singular_values
        out[f"disc{idx}"] = res.discarded_weight
    np.savez_compressed(OUT / "svd_cases_large.npz", **out)
    print("svd_cases_large")


if __name__ == "__main__" and "--svd-large" in sys.argv:
    svd_cases_large()


# Round-2 fixtures (VERDICT r1 "next" item 1): the paper's 165-qubit d=6 case
# at both truncation budgets, config 5 at every interaction distance, and more
# rows at d=6/7/8 (second seed).  Each case runs in its own process:
#     python tests/golden/make_golden.py --case <name>
ROUND2_CASES = {
    # m=165, d=6: PAPER.md:381/:388 (largest d at 165 qubits); budget 1e-24 is
    # the reference default (peak chi ~109, capacity 128), 1e-16 the paper's
    # fidelity cutoff (peak chi ~41, capacity 48)
    "stretch_m165_d6_b24": (165, 2, 6, 0.1, 1e-24, 8, 4, 0),
    "stretch_m165_d6_b16": (165, 2, 6, 0.1, 1e-16, 8, 4, 0),
    # config 5 (m=100, gamma 0.1, budget 1e-16) at the distances round 1 lacked
    "config5_m100_d1": (100, 2, 1, 0.1, 1e-16, 8, 4, 0),
    "config5_m100_d2": (100, 2, 2, 0.1, 1e-16, 8, 4, 0),
    "config5_m100_d3": (100, 2, 3, 0.1, 1e-16, 8, 4, 0),
    "config5_m100_d5": (100, 2, 5, 0.1, 1e-16, 8, 4, 0),
    # more d=6/7/8 rows (seed 1: disjoint from the round-1 seed-0 rows)
    "config5_m100_d6_s1": (100, 2, 6, 0.1, 1e-16, 8, 4, 1),
    "config5_m100_d7_s1": (100, 2, 7, 0.1, 1e-16, 8, 4, 1),
    "config5_m100_d8_s1": (100, 2, 8, 0.1, 1e-16, 8, 4, 1),
}

if __name__ == "__main__" and "--case" in sys.argv:
    _name = sys.argv[sys.argv.index("--case") + 1]
    gram_case(_name, *ROUND2_CASES[_name][:7], seed=ROUND2_CASES[_name][7])


def ops_sequences():
    """Reference results of tests/golden/ops_cases.py (apply_* / canonicalize /
    run_circuit on given states, mps.py:123-247)."""
    sys.path.insert(0, str(OUT))
    import ops_cases

    out = {}
    for name, m, budget, steps in ops_cases.cases():
        st, log = ops_cases.run(mps, ansatz, m, budget, steps)
        out[name + "_sv"] = mps.to_statevector(st)
        out[name + "_chi"] = np.array(st.bond_dims(), dtype=np.int32)
        out[name + "_discard"] = st.accumulated_discard
        out[name + "_peak"] = st.peak_chi
        out[name + "_center"] = st.ortho_center
        out[name + "_counts"] = np.array([st.gate_count_1q, st.gate_count_2q])
        out[name + "_memlog"] = np.array(log, dtype=np.int64)
    np.savez_compressed(OUT / "ops_sequences.npz", **out)
    print("ops_sequences:", len(ops_cases.cases()))


if __name__ == "__main__" and "--ops" in sys.argv:
    ops_sequences()


def experiment_config1():
    """cmd_experiment (cli.py:152-214) end to end on config 1 (m=8, d=1, 2
    layers, gamma 0.5, untruncated, 40+40 overlapping blobs (separation 1.5),
    Gaussian baseline): the
    reference's metric rows over its default C grid (cli.py:61-64) through
    its own SMO learner (learn.py:188-336)."""
    import json
    import tempfile

    from mpskernel import cli

    cfg = cli.ExperimentConfig(synthetic=cli.SyntheticSpec(n_per_class=40, separation=1.5), m=8, r=2, d=1, gamma=0.5,
                               budget=0.0, baseline=True, seed=0)
    with tempfile.TemporaryDirectory() as tmp:
        res = cli.cmd_experiment(cfg, tmp)
        K_train = np.loadtxt(f"{tmp}/gram_train.csv", delimiter=",")
        K_test = np.loadtxt(f"{tmp}/gram_test.csv", delimiter=",")
    keep = {k: res[k] for k in ("split", "rescale_params", "quantum", "best_quantum", "gaussian", "best_gaussian")}
    (OUT / "experiment_config1.json").write_text(json.dumps(keep, indent=1, sort_keys=True))
    np.savez_compressed(OUT / "experiment_config1_K.npz", K_train=K_train, K_test=K_test)
    print("experiment_config1: best AUC", res["best_quantum"]["test"]["auc"])


if __name__ == "__main__" and "--experiment" in sys.argv:
    experiment_config1()
