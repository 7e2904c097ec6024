"""Debug-build probe: average Jacobi rounds / sweeps per two-qubit SVD per config.

Needs a library built with -DMPSKQ_DEBUG_COUNTERS (pass it through MPSKQ_LIB)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np

import paper_2411_09336_b200 as P
from paper_2411_09336_b200 import _native as N
from paper_2411_09336_b200.kernel import simulate_rows

lib = N.lib()
fn = lib.mpskq_debug_counters
fn.argtypes = [C.POINTER(C.c_ulonglong)]
prev = np.zeros(3, dtype=np.uint64)
for name, (m, d, gamma, budget, n) in {
    "headline": (165, 1, 0.1, 1e-24, 512), "config2": (50, 2, 0.1, 1e-24, 256),
    "config3": (100, 4, 0.1, 1e-16, 128), "config5_d6": (100, 6, 0.1, 1e-16, 64)}.items():
    X = np.random.default_rng(0).uniform(0, 2, (n, m))
    simulate_rows(X, P.FeatureMapConfig(m, 2, d, gamma), budget)
    out = (C.c_ulonglong * 3)()
    fn(out)
    cur = np.array(list(out), dtype=np.uint64)
    r, s, sp = (cur - prev).astype(float)
    prev = cur
    print(f"{name}: {s:.0f} SVDs, {r / s:.1f} rounds/SVD, {r / sp:.2f} sweeps/SVD")
