"""Simulation device time of a config at its natural capacity (A/B of NT choices):
    MPSKQ_LIB=... python tools/ab_sim_cfg.py m d budget n cap"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2411_09336_b200 as P
from paper_2411_09336_b200.kernel import simulate_rows

m, d, budget, n, cap = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
X = np.random.default_rng(0).uniform(0, 2, (n, m))
cfg = P.FeatureMapConfig(m, 2, d, 0.1)
simulate_rows(X[:64], cfg, budget, chi_cap=cap)
ts = [simulate_rows(X, cfg, budget, chi_cap=cap).seconds * 1e3 for _ in range(2)]
print(f"m={m} d={d} n={n} cap={cap}: sim {min(ts):.1f} ms")
