"""Headline simulation time (6400 rows, capacity 4), device time of 3 runs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2411_09336_b200 as P
from paper_2411_09336_b200.kernel import simulate_rows

X = np.random.default_rng(0).uniform(0, 2, (6400, 165))
cfg = P.FeatureMapConfig(165, 2, 1, 0.1)
simulate_rows(X, cfg, 1e-24, chi_cap=4)
ts = []
for _ in range(3):
    b = simulate_rows(X, cfg, 1e-24, chi_cap=4)
    ts.append(b.seconds * 1e3)
print(f"headline sim: {min(ts):.2f} ms (runs {', '.join(f'{t:.2f}' for t in ts)})")
