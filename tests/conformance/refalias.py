"""pytest plugin: run the reference package's OWN test suite against this
package, in place (nothing is copied into the repo).

Installs ``sys.modules`` aliases before collection:
  adacluster, adacluster.{clustering, pipeline, quest, reference, tensorops,
  errors, npyio}  ->  paper_2604_18348_b200 and its modules
  adacluster.harness.*  ->  the reference's UNMODIFIED harness package
                            (baseline/_ref, installed from /root/reference),
                            whose relative imports then resolve to the
                            aliased modules -- i.e. the reference harness
                            drives the B200 package as a drop-in caller.

Used by tests/test_conformance.py as ``python -m pytest -p refalias <dir>``.
"""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
MODULES = ("clustering", "pipeline", "quest", "reference", "tensorops", "errors", "npyio")


def _harness_dir() -> Path | None:
    for cand in (os.environ.get("AC_REF_HARNESS"),
                 ROOT / "baseline" / "_ref" / "adacluster" / "harness",
                 "/root/reference/pkg/src/adacluster/harness"):
        if cand and (Path(cand) / "__init__.py").exists():
            return Path(cand)
    return None


def install() -> None:
    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    pkg = importlib.import_module("paper_2604_18348_b200")
    sys.modules["adacluster"] = pkg
    for m in MODULES:
        sys.modules[f"adacluster.{m}"] = importlib.import_module(f"paper_2604_18348_b200.{m}")
    hd = _harness_dir()
    if hd is not None:
        spec = importlib.util.spec_from_file_location(
            "adacluster.harness", hd / "__init__.py", submodule_search_locations=[str(hd)])
        mod = importlib.util.module_from_spec(spec)
        sys.modules["adacluster.harness"] = mod
        spec.loader.exec_module(mod)


def pytest_configure(config):
    install()
