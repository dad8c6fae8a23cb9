"""INTEGRATION.md's ctypes binding, dropped into a scratch copy of the
reference package (only where /root/reference exists, i.e. the build
container): the stub imports what it needs from pbbem, marshals a real
pbbem problem into hobi_create's C signature, and without a GPU gets the
library's "no CUDA device" error back -- i.e. the binding a maintainer would
add runs as written up to the device."""
import os
import re
import shutil
import sys

import pytest

from conftest import ROOT

REF = "/root/reference/pkg/src/pbbem"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
def test_integration_stub_binds_reference_objects(tmp_path):
    from paper_1301_5914_b200 import _native as N

    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = re.search(r"```python\n(# pbbem/_b200\.py.*?)```", text, flags=re.S).group(1)
    block = block.replace('C.CDLL("libhobi.so")', f'C.CDLL({N.LIB_PATH!r})')
    pkg = tmp_path / "pbbem"
    shutil.copytree(REF, pkg)
    (pkg / "_b200.py").write_text(block)
    sys.path.insert(0, str(tmp_path))
    try:
        for mod in [m for m in sys.modules if m == "pbbem" or m.startswith("pbbem.")]:
            del sys.modules[mod]
        import pbbem
        from pbbem._b200 import B200Operator

        mesh = pbbem.icosahedral_sphere(1, radius=2.0)
        params = pbbem.PhysicalParams(eps1=1.0, eps2=80.0, kappa=0.1257)
        charges = pbbem.ChargeSystem(positions=[[0.0, 0.0, 0.0]], charges=[1.0])
        config = pbbem.SolverConfig(workers=1)
        problem = pbbem.discretize(mesh, params, charges, config)
        if N.device_count() > 0:
            with B200Operator(problem, config) as op:
                import numpy as np

                u = np.random.default_rng(0).standard_normal(problem.n_unknowns)
                assert np.allclose(op(u), pbbem.matvec_hobi(problem, u), rtol=1e-10, atol=1e-12)
        else:
            with pytest.raises(RuntimeError, match="CUDA|device"):
                B200Operator(problem, config)
    finally:
        sys.path.remove(str(tmp_path))
        for mod in [m for m in sys.modules if m == "pbbem" or m.startswith("pbbem.")]:
            del sys.modules[mod]
