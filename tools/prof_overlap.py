"""Profiling driver: simulate N headline rows, then run the train-kernel
overlap `reps` times (the launch to profile is the last one)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

import paper_2411_09336_b200 as P
from paper_2411_09336_b200.kernel import simulate_rows
from paper_2411_09336_b200.mps import overlap_matrix

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--m", type=int, default=165)
ap.add_argument("--d", type=int, default=1)
ap.add_argument("--budget", type=float, default=1e-24)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--sim-only", action="store_true")
a = ap.parse_args()
cfg = P.FeatureMapConfig(a.m, 2, a.d, 0.1)
X = np.random.default_rng(0).uniform(0, 2, (a.n, a.m))
b = simulate_rows(X, cfg, a.budget)
torch.cuda.synchronize()
if a.sim_only:
    for _ in range(a.reps):
        b = simulate_rows(X, cfg, a.budget)
else:
    for _ in range(a.reps):
        K = overlap_matrix(b, b, "train")
torch.cuda.synchronize()
print("ok", b.chi_cap, len(b))
