"""Run the REFERENCE's own test suite (pkg/tests, 176 tests) against this
package: ``qttfem`` and its submodules are aliased to ``paper_2501_07778_b200``
(the drop-in claim of SURVEY §8(b)), except ``qttfem.oracle`` -- the
conforming sparse FEM the reference tests use as ground truth (out of scope,
stays on the CPU) -- which is the reference's own module, imported with its
relative imports resolved to OUR element / material / topology modules.

The reference is not copied into the repository: ``baseline/_ref`` (git
ignored, travels with gpurun) holds the offline pip install of
/root/reference plus a copy of pkg/tests, made in the development container:

    python -m pip install --no-index --no-build-isolation --no-deps \\
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>
    mkdir -p baseline/_ref/pkg_tests && cp /root/reference/pkg/tests/*.py baseline/_ref/pkg_tests/

Usage (on the GPU box): python tools/run_reference_suite.py [pytest args]
"""
import importlib
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
sys.path.insert(0, ROOT)

import paper_2501_07778_b200 as pkg  # noqa: E402

sys.modules["qttfem"] = pkg
for name in ("ttcore", "indexing", "element", "material", "mesh", "topology", "assembly", "coupling",
             "solver"):
    mod = importlib.import_module(f"paper_2501_07778_b200.{name}")
    sys.modules[f"qttfem.{name}"] = mod
    setattr(pkg, name, mod)
spec = importlib.util.spec_from_file_location("qttfem.oracle", os.path.join(REF, "qttfem", "oracle.py"),
                                              submodule_search_locations=None)
oracle = importlib.util.module_from_spec(spec)
oracle.__package__ = "qttfem"
sys.modules["qttfem.oracle"] = oracle
spec.loader.exec_module(oracle)
pkg.oracle = oracle

import pytest  # noqa: E402

args = sys.argv[1:] or ["-q", "-rfE", "--tb=line"]
sys.exit(pytest.main([os.path.join(REF, "pkg_tests"), "-p", "no:cacheprovider", "-p", "no:randomly"] + args))
