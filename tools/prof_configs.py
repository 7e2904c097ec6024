"""Profiling driver for the secondary configurations: simulate N rows of a
named config (capacity fixed) and run its train-kernel overlap once, so an
ncu capture filtered to one kernel sees exactly one launch of it.

    python tools/prof_configs.py CONFIG [--n N] [--sim-only]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2411_09336_b200 as P  # noqa: E402
from paper_2411_09336_b200.kernel import simulate_rows  # noqa: E402
from paper_2411_09336_b200.mps import overlap_matrix  # noqa: E402

CONFIGS = {  # name: (m, d, gamma, budget, chi_cap)
    "c5_d2_cap8": (100, 2, 0.1, 1e-16, 8),
    "c2_cap12": (50, 2, 0.1, 1e-24, 12),
    "c3_cap24": (100, 4, 0.1, 1e-16, 24),
    "c5_d6_cap48": (100, 6, 0.1, 1e-16, 48),
    "c5_d8_cap96": (100, 8, 0.1, 1e-16, 96),
    "s6_b24_cap128": (165, 6, 0.1, 1e-24, 128),
}

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=sorted(CONFIGS))
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--sim-only", action="store_true")
a = ap.parse_args()
m, d, gamma, budget, cap = CONFIGS[a.config]
cfg = P.FeatureMapConfig(m, 2, d, gamma)
X = np.random.default_rng(0).uniform(0, 2, (a.n, m))
b = simulate_rows(X, cfg, budget, chi_cap=cap)
torch.cuda.synchronize()
if not a.sim_only:
    K = overlap_matrix(b, b, "train")
    torch.cuda.synchronize()
print("ok", a.config, b.chi_cap, len(b), int(b.bond_dims().max()))
