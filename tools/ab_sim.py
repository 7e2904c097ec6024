"""Same-box A/B of the simulator on one wave of states at a forced capacity:
    MPSKQ_LIB=... python tools/ab_sim.py m d budget n cap"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2411_09336_b200 as P
from paper_2411_09336_b200.kernel import simulate_rows

m, d, budget, n, cap = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
X = np.random.default_rng(0).uniform(0, 2, (n, m))
cfg = P.FeatureMapConfig(m, 2, d, 0.1)
simulate_rows(X[:8], cfg, budget, chi_cap=cap)
torch.cuda.synchronize()
t = time.time()
b = simulate_rows(X, cfg, budget, chi_cap=cap)
torch.cuda.synchronize()
print(f"m={m} d={d} budget={budget} n={n} cap={cap}: {time.time() - t:.2f} s, peak {int(b.peak.max())}")
