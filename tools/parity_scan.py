"""At-scale parity scan: GPU simulation of N headline rows vs the CPU oracle
(bitwise the reference, tests/test_oracle.py) on every row, plus K on a random
sample of pairs.  Oracle work runs in a host process pool.

    python tools/parity_scan.py [--rows 6400] [--pairs 2000] [--config headline]
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

CONFIGS = {
    "headline": (165, 1, 0.1, 1e-24),
    "config2": (50, 2, 0.1, 1e-24),
    "config3": (100, 4, 0.1, 1e-16),
}


def _oracle_row(args):
    x, m, d, gamma, budget = args
    from oracle import mps_oracle as O

    st = O.simulate_row(x, m, 2, d, gamma, budget)
    return st.bond_dims(), st.sites, st.discard


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=6400)
    ap.add_argument("--pairs", type=int, default=2000)
    ap.add_argument("--config", default="headline")
    a = ap.parse_args()
    m, d, gamma, budget = CONFIGS[a.config]
    X = np.random.default_rng(0).uniform(0.0, 2.0, (a.rows, m))

    t0 = time.time()
    cores = len(os.sched_getaffinity(0))
    with mp.get_context("fork").Pool(cores) as pool:
        ref = pool.map(_oracle_row, [(x, m, d, gamma, budget) for x in X], chunksize=8)
    t_oracle = time.time() - t0

    import torch

    import paper_2411_09336_b200 as P
    from oracle import mps_oracle as O

    cfg = P.FeatureMapConfig(m, 2, d, gamma)
    batch = P.simulate_dataset(X, cfg, budget=budget)
    K = P.compute_gram(batch, batch, "train").entries
    torch.cuda.synchronize()
    chi = batch.bond_dims()
    ref_chi = [r[0] for r in ref]
    mismatch = [i for i in range(a.rows) if chi[i].tolist() != ref_chi[i]]
    disc = batch.discard.cpu().numpy()
    rng = np.random.default_rng(1)
    pairs = rng.integers(0, a.rows, size=(a.pairs, 2))
    pairs = pairs[pairs[:, 0] != pairs[:, 1]]
    err = [abs(K[i, j] - abs(O.overlap(ref[i][1], ref[j][1])) ** 2) for i, j in pairs]
    out = {
        "config": a.config, "m": m, "d": d, "gamma": gamma, "budget": budget, "rows": a.rows,
        "bond_dim_mismatched_states": len(mismatch), "mismatched_indices": mismatch[:20],
        "max_abs_discard_diff": float(np.max(np.abs(disc - np.array([r[2] for r in ref])))),
        "sampled_pairs": int(len(pairs)), "max_abs_K_err": float(np.max(err)),
        "mean_abs_K_err": float(np.mean(err)),
        "diag_all_one": bool(np.all(np.diag(K) == 1.0)), "symmetric": bool(np.array_equal(K, K.T)),
        "oracle_seconds": t_oracle, "oracle_cores": cores,
    }
    print(json.dumps(out))
    Path("gpurun_out").mkdir(exist_ok=True)
    Path(f"gpurun_out/parity_scan_{a.config}.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
