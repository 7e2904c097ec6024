"""Downstream parity: the reference's own experiment flow
(cli.cmd_experiment, cli.py:152-214: split, rescale, train/test kernels
through run_distributed, SMO SVM over the default C grid, AUC/accuracy
metrics, learn.py:188-336) run on the GPU kernels must give the reference's
metric rows exactly.

The reference's learn/cli come from baseline/_ref (the unmodified reference,
pip-installed there, git-ignored; it travels to the GPU box with the
snapshot).  The test skips when it is absent."""

import json
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

REF = ROOT / "baseline" / "_ref" / "mpskernel"


@pytest.mark.skipif(not REF.exists(), reason="reference not installed in baseline/_ref")
def test_cmd_experiment_metrics_match_reference(tmp_path):
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "refshim" / "run_experiment.py"), str(tmp_path)],
                         capture_output=True, text=True, check=True, cwd=str(ROOT))
    res = json.loads(out.stdout.strip().splitlines()[-1])
    want = golden("experiment_config1.json")
    assert res["split"] == want["split"]
    for key in ("quantum", "best_quantum", "gaussian", "best_gaussian"):
        assert res[key] == want[key], key  # C, n_support, train/test AUC, accuracy, ... identical
    Kg = golden("experiment_config1_K.npz")
    K_train = np.loadtxt(tmp_path / "gram_train.csv", delimiter=",")
    K_test = np.loadtxt(tmp_path / "gram_test.csv", delimiter=",")
    assert np.abs(K_train - Kg["K_train"]).max() < 1e-10
    assert np.abs(K_test - Kg["K_test"]).max() < 1e-10
    # the reference's report counters, from the GPU run
    n_tr = len(want["split"]["train_indices"])
    n_te = len(want["split"]["test_indices"])
    assert res["report"]["n_inner_products"] == n_tr * (n_tr - 1) // 2 + n_te * n_tr
