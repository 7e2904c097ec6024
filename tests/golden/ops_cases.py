"""Deterministic gate/canonicalize sequences on given states, shared by
make_golden.py (run against the reference) and tests/test_gpu_ops.py (run
against the GPU drop-in): apply_one_qubit / apply_two_qubit with Haar-random
unitaries and both absorb sides, apply_gate (incl. reversed qubit order),
canonicalize to random centers and run_circuit continuing a given state
(reference mps.py:123-247)."""

from __future__ import annotations

import numpy as np


def _haar(rng, n):
    z = rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))
    q, r = np.linalg.qr(z)
    return q * (np.diag(r) / np.abs(np.diag(r)))


def cases():
    """(name, m, budget, steps); a step is a tuple (op, args...)."""
    out = []
    for idx, (m, budget, n_steps) in enumerate([(6, 1e-24, 40), (8, 1e-12, 60), (7, 0.0, 50), (10, 1e-6, 80)]):
        rng = np.random.default_rng(1000 + idx)
        steps = [("gate", "H", (q,), None) for q in range(m)]
        for _ in range(n_steps):
            r = rng.random()
            if r < 0.2:
                steps.append(("u1", int(rng.integers(m)), _haar(rng, 2)))
            elif r < 0.6:
                steps.append(("u2", int(rng.integers(m - 1)), _haar(rng, 4), "left" if rng.random() < 0.5 else "right"))
            elif r < 0.75:
                steps.append(("can", int(rng.integers(m))))
            elif r < 0.9:
                q = int(rng.integers(m - 1))
                qs = (q + 1, q) if rng.random() < 0.5 else (q, q + 1)
                steps.append(("gate", "RXX", qs, float(rng.uniform(-3, 3))))
            else:
                steps.append(("gate", "RZ", (int(rng.integers(m)),), float(rng.uniform(-3, 3))))
        out.append((f"ops{idx}_m{m}", m, budget, steps))
    return out


def run(mod, ansatz, m, budget, steps, circuit_tail=True):
    """Apply `steps` with module `mod` (reference mpskernel.mps or the drop-in)
    to init_state(m); then run_circuit of a feature circuit on the result."""
    st = mod.init_state(m, "zero", trunc_budget_per_gate=budget)
    for s in steps:
        if s[0] == "u1":
            mod.apply_one_qubit(st, s[1], s[2])
        elif s[0] == "u2":
            mod.apply_two_qubit(st, s[1], s[2], absorb=s[3])
        elif s[0] == "can":
            mod.canonicalize(st, s[1])
        else:
            mod.apply_gate(st, ansatz.Gate(s[1], s[2], s[3]))
    log = []
    if circuit_tail:
        cfg = ansatz.FeatureMapConfig(m, 1, 2, 0.7)
        x = np.random.default_rng(m).uniform(0.0, 2.0, m)
        mod.run_circuit(st, ansatz.encode_circuit(x, cfg), memory_log=log)
    return st, log
