"""pytest plugin: run the REFERENCE's own test suite against the GPU drop-in.

    PYTHONPATH=tools/refshim:baseline/_ref/tests python -m pytest -p refshim_plugin baseline/_ref/tests

`baseline/_ref` holds the unmodified reference (pip-installed from
/root/reference/pkg, git-ignored, travels to the GPU box) plus a copy of its
tests.  Before any test imports `mpskernel`, this plugin assembles a package
of that name in which every public name the drop-in `paper_2411_09336_b200`
defines replaces the reference's:

* `mpskernel.ansatz / .tensor / .mps / .kernel`: the reference module's
  source is executed first (so names the drop-in does not define keep the
  reference's definition), then every public name the drop-in also defines
  is replaced by the drop-in's (GPU) implementation;
* `mpskernel.learn / .cli` (SVM, CLI: downstream of K, out of the hot
  path) are the reference's, and their relative imports resolve to the
  merged modules above, so `cmd_experiment` / `cmd_gram` / `cmd_benchmark`
  run on the GPU kernels.

Which names came from where is written to gpurun_out/refshim_names.json.
"""

from __future__ import annotations

import importlib
import importlib.util
import json
import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
REF = ROOT / "baseline" / "_ref" / "mpskernel"
MERGED = ("tensor", "ansatz", "mps", "kernel")
REFERENCE_ONLY = ("learn", "cli")


def _exec_ref(name: str) -> types.ModuleType:
    full = f"mpskernel.{name}"
    spec = importlib.util.spec_from_file_location(full, REF / f"{name}.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules[full] = mod
    spec.loader.exec_module(mod)
    return mod


def install() -> dict:
    if not REF.exists():
        raise RuntimeError(f"{REF} missing: pip install the reference into baseline/_ref first")
    sys.path.insert(0, str(ROOT))
    pkg = types.ModuleType("mpskernel")
    pkg.__path__ = [str(REF)]
    pkg.__file__ = str(REF / "__init__.py")
    pkg.__package__ = "mpskernel"
    sys.modules["mpskernel"] = pkg
    report = {}
    for name in MERGED:
        mod = _exec_ref(name)
        ours = importlib.import_module(f"paper_2411_09336_b200.{name}")
        replaced, kept = [], []
        for attr in sorted(vars(mod)):
            if attr.startswith("__"):
                continue
            val = getattr(mod, attr)
            if isinstance(val, types.ModuleType) or getattr(val, "__module__", None) not in (mod.__name__, None):
                continue  # imports of the reference module (numpy, dataclasses, sibling modules)
            if hasattr(ours, attr):
                setattr(mod, attr, getattr(ours, attr))
                replaced.append(attr)
            else:
                kept.append(attr)
        setattr(pkg, name, mod)
        report[name] = {"drop_in": replaced, "reference": kept}
    for name in REFERENCE_ONLY:
        setattr(pkg, name, _exec_ref(name))
        report[name] = {"drop_in": [], "reference": ["(whole module)"]}
    src = (REF / "__init__.py").read_text()
    exec(compile(src, str(REF / "__init__.py"), "exec"), pkg.__dict__)
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / "refshim_names.json").write_text(json.dumps(report, indent=1))
    return report


install()
