"""cmd_experiment (reference cli.py:152-214) with the reference's own CLI and
SMO learner on top of the GPU drop-in (refshim_plugin assembles `mpskernel`
from the drop-in's hot path + the reference's learn/cli).  Prints the metric
rows as JSON; tests/test_gpu_downstream.py compares them with the
reference's (tests/golden/experiment_config1.json).

    python tools/refshim/run_experiment.py OUT_DIR
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import refshim_plugin  # noqa: E402,F401  (installs the merged `mpskernel`)

from mpskernel import cli  # noqa: E402

cfg = cli.ExperimentConfig(synthetic=cli.SyntheticSpec(n_per_class=40, separation=1.5), m=8, r=2, d=1, gamma=0.5,
                           budget=0.0, baseline=True, seed=0)
res = cli.cmd_experiment(cfg, sys.argv[1])
print(json.dumps({k: res[k] for k in ("split", "rescale_params", "quantum", "best_quantum", "gaussian",
                                      "best_gaussian", "report")}))
