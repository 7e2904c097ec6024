"""Overlap time of the same states at several forced capacities (layout A/B)."""
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
import torch

import paper_2411_09336_b200 as P
from paper_2411_09336_b200.kernel import simulate_rows
from paper_2411_09336_b200.mps import overlap_matrix

for (m, d, budget, n, caps) in [(100, 4, 1e-16, 400, [24, 32]), (100, 5, 1e-16, 300, [32, 48]),
                                 (100, 6, 1e-16, 300, [48, 64, 96]), (100, 7, 1e-16, 300, [64, 96]),
                                 (100, 8, 1e-16, 148, [96, 128])]:
    X = np.random.default_rng(0).uniform(0, 2, (n, m))
    cfg = P.FeatureMapConfig(m, 2, d, 0.1)
    for cap in caps:
        b = simulate_rows(X, cfg, budget, chi_cap=cap)
        overlap_matrix(b, b, "train")
        torch.cuda.synchronize()
        t = time.time()
        overlap_matrix(b, b, "train")
        torch.cuda.synchronize()
        print(f"d={d} n={n} cap={cap}: overlap {1e3 * (time.time() - t):.1f} ms", flush=True)
