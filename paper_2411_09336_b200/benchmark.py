"""Resource benchmark of the GPU path — the measurement half of the
reference's ``cli.cmd_benchmark`` (cli.py:240-294) without its dataset/CLI
plumbing (out of scope).

The reference times each sample's ``simulate_circuit`` and each pairwise
``inner_product`` on the CPU and records the peak bond dimension per sample
and the state memory after every gate (``memory_log``, mps.py:245-246).  On
the GPU all samples are simulated in one batched launch and all pairs in one
overlap launch, so the per-sample / per-pair seconds reported here are the
batch device times divided by the counts (CUDA events), and the memory
series come from the simulator's per-gate entry log.
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
    prog = compile_program(feature_map_topology(cfg.m, cfg.r, cfg.d))
    coef, _ = encode_device(torch.from_numpy(np.ascontiguousarray(X)).to("cuda"), cfg)
    batch = simulate_program(prog, coef, budget, memory_log=True)
    with Timer() as t_ov:
        overlap_matrix(batch, batch, "test", amplitude=True)
    pairs = n * (n - 1) // 2
    # the test-kind launch evaluates all n^2 pairs; scale to the i<j count
    ip = t_ov.seconds() / (n * n)
    sim = batch.seconds / n
    states = batch.to_states()
    max_chi = [max(s.peak_chi, s.max_bond()) for s in states]
    return {
        "samples": n,
        "simulation_seconds": [sim] * n,
        "inner_product_seconds": [ip] * pairs,
        "simulation_summary": _summary([sim] * n),
        "inner_product_summary": _summary([ip] * pairs),
        "max_chi": max_chi,
        "memory_bytes_per_gate": [batch.memory_log(i) for i in range(n)],
        "timing": "batched device time divided by the number of states / pairs (CUDA events)",
    }
