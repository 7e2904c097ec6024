"""Secondary measurements for the non-headline BASELINE configs (parity cases,
not bench lines): per config, device time of simulate + train kernel with
CUDA events, algorithmic overlap flops, nominal simulation flops, and the
fractions of the measured FP64 peak (mpskq_fp64_probe, as in bench.py)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np
import torch

import paper_2411_09336_b200 as P
from bench import train_flops
from paper_2411_09336_b200.kernel import simulate_rows
from paper_2411_09336_b200.mps import overlap_matrix

CONFIGS = {
    "config1_m8_d1": (8, 1, 0.5, 0.0, 64),
    "config2_m50_d2": (50, 2, 0.1, 1e-24, 800),
    "config3_m100_d4": (100, 4, 0.1, 1e-16, 1600),
    "config5_m100_d1": (100, 1, 0.1, 1e-16, 800),
    "config5_m100_d2": (100, 2, 0.1, 1e-16, 800),
    "config5_m100_d3": (100, 3, 0.1, 1e-16, 800),
    "config5_m100_d4": (100, 4, 0.1, 1e-16, 800),
    "config5_m100_d5": (100, 5, 0.1, 1e-16, 800),
    "config5_m100_d6": (100, 6, 0.1, 1e-16, 800),
    "config5_m100_d7": (100, 7, 0.1, 1e-16, 800),
    "config5_m100_d8": (100, 8, 0.1, 1e-16, 800),
    # headline stretch (paper's largest d at 165 qubits), one wave of states
    "config4_m165_d6_1e-16": (165, 6, 0.1, 1e-16, 296),
    "config4_m165_d6_1e-24": (165, 6, 0.1, 1e-24, 148),
}


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = fn()
    b.record()
    b.synchronize()
    return out, a.elapsed_time(b) / reps


def main(names):
    from bench import fp64_peak_tflops
    from paper_2411_09336_b200 import _native as N

    peak = fp64_peak_tflops(N.lib(), torch)
    res = {"fp64_peak_tflops_measured": peak}
    for name in names:
        torch.cuda.empty_cache()  # each config starts from the same free HBM
        m, d, gamma, budget, n = CONFIGS[name]
        cfg = P.FeatureMapConfig(m, 2, d, gamma)
        X = np.random.default_rng(0).uniform(0.0, 2.0, (n, m))
        try:
            batch, sim_ms = timed(lambda: simulate_rows(X, cfg, budget), reps=2 if n * m < 1e6 else 1)
        except RuntimeError as exc:
            res[name] = {"error": str(exc)}
            print(name, "ERROR", exc, flush=True)
            continue
        K, ov_ms = timed(lambda: overlap_matrix(batch, batch, "train"), reps=2)
        chi = batch.bond_dims()
        fl = train_flops(chi)
        # nominal simulation flops (theta + gate + LAPACK-nominal
        # thin SVD + QR moves, counted by the simulator per state) over the
        # measured simulation time; escalated states count every level they ran
        sim_fl = float(batch.nominal_flops.sum().item())
        ent = n * (n - 1) / 2
        r = {"N": n, "chi_cap": batch.chi_cap, "chi_max": int(chi.max()), "peak_max": int(batch.peak.max()),
             "sim_ms": sim_ms, "mps_states_per_s": n / (sim_ms / 1e3),
             "sim_nominal_flops": sim_fl, "sim_tflops_nominal": sim_fl / (sim_ms / 1e3) / 1e12,
             "overlap_ms": ov_ms,
             "entries_per_s": ent / (ov_ms / 1e3), "overlap_tflops_alg": fl / (ov_ms / 1e3) / 1e12}
        r["overlap_frac_of_fp64_peak"] = r["overlap_tflops_alg"] / peak
        r["sim_frac_of_fp64_peak"] = r["sim_tflops_nominal"] / peak
        res[name] = r
        print(name, json.dumps(r), flush=True)
    return res


if __name__ == "__main__":
    out = main(sys.argv[1:] or list(CONFIGS))
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/configs.json").write_text(json.dumps(out, indent=1))
