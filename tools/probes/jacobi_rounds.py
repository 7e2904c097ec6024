"""Debug-build probe: Jacobi rounds / sweeps per two-qubit SVD and the SM-cycle
split of the simulator's phases, per config.

Needs a library built with -DMPSKQ_DEBUG_COUNTERS, passed through MPSKQ_LIB:
    python -c "from paper_2411_09336_b200 import build as b; \\
               b.build(out='ab/libmpskq_dbg.so', defines=('MPSKQ_DEBUG_COUNTERS',))"
    MPSKQ_LIB=ab/libmpskq_dbg.so python tools/probes/jacobi_rounds.py [names...]
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np

import paper_2411_09336_b200 as P
from paper_2411_09336_b200 import _native as N
from paper_2411_09336_b200.kernel import simulate_rows

PHASES = ["theta build", "QRCP + R^H", "Jacobi", "norms + truncation", "C-side write + replay",
          "Q application", "W-side write", "QR moves"]
CONFIGS = {
    "headline": (165, 1, 0.1, 1e-24, 512), "config2": (50, 2, 0.1, 1e-24, 256),
    "config3": (100, 4, 0.1, 1e-16, 128), "config5_d6": (100, 6, 0.1, 1e-16, 64),
    "config5_d8": (100, 8, 0.1, 1e-16, 32), "m165_d6_1e-24": (165, 6, 0.1, 1e-24, 16),
}

lib = N.lib()
fn = lib.mpskq_debug_counters
fn.argtypes = [C.POINTER(C.c_ulonglong)]
fc = getattr(lib, "mpskq_debug_cycles", None)
if fc is not None:
    fc.argtypes = [C.POINTER(C.c_ulonglong)]
prev = np.zeros(3, dtype=np.uint64)
prevc = np.zeros(8, dtype=np.uint64)
for name in sys.argv[1:] or list(CONFIGS)[:4]:
    m, d, gamma, budget, n = CONFIGS[name]
    X = np.random.default_rng(0).uniform(0, 2, (n, m))
    simulate_rows(X, P.FeatureMapConfig(m, 2, d, gamma), budget)
    out = (C.c_ulonglong * 3)()
    fn(out)
    cur = np.array(list(out), dtype=np.uint64)
    r, s, sp = (cur - prev).astype(float)
    prev = cur
    line = f"{name}: {s:.0f} SVDs, {r / s:.1f} rounds/SVD, {r / sp:.2f} sweeps/SVD"
    if fc is not None:
        oc = (C.c_ulonglong * 8)()
        fc(oc)
        curc = np.array(list(oc), dtype=np.uint64)
        dc = (curc - prevc).astype(float)
        prevc = curc
        tot = dc.sum() or 1.0
        line += " | " + ", ".join(f"{p} {100 * v / tot:.0f}%" for p, v in zip(PHASES, dc))
    print(line, flush=True)
