"""The reference's own host-only tests (test_ansatz.py: feature map, layer
scheduling, SWAP routing) against the drop-in through the import shim
(tools/refshim/refshim_plugin.py) — CPU only.  The GPU box runs the whole
reference suite the same way (tools/gpu/run_reference_suite.sh)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF = ROOT / "baseline" / "_ref"


@pytest.mark.skipif(not (REF / "tests" / "test_ansatz.py").exists(), reason="reference not installed in baseline/_ref")
def test_reference_ansatz_suite_passes_through_the_shim():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(ROOT / "tools" / "refshim"), str(REF / "tests")]))
    out = subprocess.run([sys.executable, "-m", "pytest", "-p", "refshim_plugin", str(REF / "tests" / "test_ansatz.py"),
                          "-q", "-p", "no:cacheprovider"], capture_output=True, text=True, cwd=str(ROOT), env=env,
                         timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert " passed" in out.stdout and "failed" not in out.stdout
