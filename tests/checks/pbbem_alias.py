"""pytest plugin (-p pbbem_alias): `import pbbem[.module]` resolves to this
repo's package, so the reference's own test files exercise the B200 package
unchanged.  Used only by tests/checks/reference_suite.py."""

import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_1301_5914_b200 as _pkg  # noqa: E402

sys.modules["pbbem"] = _pkg
for _name in ("solver", "mesh", "quadrature", "kirkwood", "report", "cli", "kernels", "geometry"):
    sys.modules["pbbem." + _name] = importlib.import_module("paper_1301_5914_b200." + _name)
