"""Per-state bond-dimension diff of the GPU simulation against a reference
fixture (tests/golden/<name>.npz): which states / bonds differ, peaks and
discards.  python tools/diag_fixture.py stretch_m165_d6_b24 [--lib path]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2411_09336_b200 as P  # noqa: E402

name = sys.argv[1]
g = np.load(Path(__file__).resolve().parent.parent / "tests" / "golden" / f"{name}.npz")
cfg = P.FeatureMapConfig(int(g["m"]), int(g["r"]), int(g["d"]), float(g["gamma"]))
budget = float(g["budget"])
for split in ("train", "test"):
    X = g["X"] if split == "train" else g["X_test"]
    b = P.simulate_dataset(X, cfg, budget=budget)
    chi = b.bond_dims()
    ref = g[f"{split}_chi"]
    peak = b.peak.cpu().numpy()
    disc = b.discard.cpu().numpy()
    print(split, "cap", b.chi_cap)
    for i in range(len(X)):
        d = np.nonzero(chi[i] != ref[i])[0]
        print(f"  row {i}: peak {peak[i]} ref {g[split + '_peak'][i]}  disc {disc[i]:.6e} ref {g[split + '_discard'][i]:.6e}"
              f"  differing bonds {len(d)}" + (f" e.g. {[(int(k), int(chi[i, k]), int(ref[i, k])) for k in d[:6]]}" if len(d) else ""))
