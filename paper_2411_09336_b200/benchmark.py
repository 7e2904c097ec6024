"""Resource benchmark of the GPU path — the measurement half of the
reference's ``cli.cmd_benchmark`` (cli.py:240-294) without its dataset/CLI
plumbing (out of scope).

Like the reference, every sample's simulation and every pairwise inner
product is timed on its own: one single-state simulation launch per sample
and one single-pair overlap launch per pair, each bracketed by CUDA events
on the launching stream (device latency of one unit, not a batch time
divided by the count).  The peak bond dimension per sample and the state
memory after every gate (``memory_log``, mps.py:245-246) come from the
simulator's per-gate entry log.
"""

from __future__ import annotations

import numpy as np
import torch

from ._device import Timer
from .ansatz import FeatureMapConfig, feature_map_topology
from .kernel import _check_rows, encode_device
from .mps import DEFAULT_TRUNC_BUDGET, compile_program, overlap_matrix, simulate_program


def _summary(values) -> dict:
    q1, med, q3 = np.percentile(values, [25, 50, 75])
    return {"median": float(med), "q1": float(q1), "q3": float(q3)}


def benchmark_rows(X, cfg: FeatureMapConfig, budget: float = DEFAULT_TRUNC_BUDGET) -> dict:
    """cmd_benchmark's payload (minus 'config') for the feature rows X."""
    X = _check_rows(X, cfg.m)
    n = X.shape[0]
    if n < 2:
        raise ValueError("benchmark needs at least 2 samples")
    # encode_circuit's row checks (ansatz.py:121-124)
    if not np.all(np.isfinite(X)):
        raise ValueError("features must be finite")
    if np.any((X < 0.0) | (X > 2.0)):
        raise ValueError("features must lie in [0, 2]; rescale the data first")
    prog = compile_program(feature_map_topology(cfg.m, cfg.r, cfg.d))
    coef, bad = encode_device(torch.from_numpy(np.ascontiguousarray(X)).to("cuda"), cfg)
    if int(bad.item()) != 0:
        raise ValueError("features must lie in [0, 2]; rescale the data first")
    # warm the program / capacity hint so the per-sample launches are steady
    simulate_program(prog, coef[:1], budget)
    states, sim_times = [], []
    for i in range(n):
        with Timer() as t:
            b = simulate_program(prog, coef[i : i + 1], budget, memory_log=True)
        sim_times.append(t.seconds())
        states.append(b)
    cap = max(b.chi_cap for b in states)
    ip_times = []
    for i in range(n):
        for j in range(i + 1, n):
            a, k = states[i], states[j]
            if a.chi_cap != cap or k.chi_cap != cap:  # one layout per pair launch
                from .mps import MpsBatch

                a = a if a.chi_cap == cap else MpsBatch.from_states(a.to_states(), cap)
                k = k if k.chi_cap == cap else MpsBatch.from_states(k.to_states(), cap)
                states[i], states[j] = a, k
            with Timer() as t:
                overlap_matrix(a, k, "test", amplitude=True)
            ip_times.append(t.seconds())
    single = [b[0] for b in states]
    return {
        "samples": n,
        "simulation_seconds": sim_times,
        "inner_product_seconds": ip_times,
        "simulation_summary": _summary(sim_times),
        "inner_product_summary": _summary(ip_times),
        "max_chi": [max(s.peak_chi, s.max_bond()) for s in single],
        "memory_bytes_per_gate": [b.memory_log(0) for b in states],
        "timing": "per sample / per pair: one launch each, CUDA events on the launching stream",
    }
