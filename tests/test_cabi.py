"""The C-ABI library loads on CPU and exports every symbol include/hobi.h
declares (no compute calls without a GPU); the product refuses to run
without a device instead of falling back to the CPU."""

import os
import sys
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1301_5914_b200 import _native as N


def _declared():
    text = open(os.path.join(ROOT, "include", "hobi.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hobi_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_expected_entry_points():
    names = _declared()
    for must in ("hobi_create", "hobi_matvec", "hobi_matvec_device", "hobi_matvec_rows", "hobi_rhs",
                 "hobi_energy", "hobi_gmres", "hobi_comm_init", "hobi_destroy", "hobi_bench"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = N.load()
    for name in _declared():
        assert hasattr(lib, name), name
        assert name in N.SIGNATURES, f"{name} has no ctypes signature"
    assert set(N.SIGNATURES) <= set(_declared())
    assert lib.hobi_abi_version() == 1


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_default_sweep_executes_the_documented_instruction_mix():
    """bench.py's FP64_INSTR_PER_PAIR and DESIGN.md's 24 DFMA + 12 DMUL + 7 DADD
    are the SASS of the default sweep variants: step_R7_minb2_unroll3 (7
    targets x 3 unrolled sources = 21 pairs per loop body, nothing else FP64)
    and step_R4_minb3_unroll2 (8 pairs), used when a row range leaves a long
    remainder past the 768-row tiles."""
    import subprocess

    import bench

    internal = open(os.path.join(ROOT, "paper_1301_5914_b200", "csrc", "hobi_internal.cuh")).read()
    assert re.search(r"int sweep_variant = 22;.*step_R7_minb2_unroll3", internal)
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", N.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    # unroll 3 over 64-source tiles: a 21-pair loop body plus a 7-pair tail (28 in the function)
    for frag, pairs, r in (("sweep_kernelILi1ELb1ELb0ELi7ELi2ELi3ELb1E", 28, 7),
                           ("sweep_kernelILi1ELb1ELb0ELi4ELi3ELi2ELb1E", 8, 4)):
        body, on = [], False
        for line in out.stdout.splitlines():
            if "Function : " in line:
                on = frag in line
            elif on:
                body.append(line)
        sass = "\n".join(body)
        counts = {op: len(re.findall(r"\b" + op + r"\b", sass)) for op in ("DFMA", "DMUL", "DADD")}
        # + two DMULs per target row when an item stores its acc2 partial (the n'z / Ap scale)
        assert counts == {"DFMA": 24 * pairs, "DMUL": 12 * pairs + 2 * r, "DADD": 7 * pairs}, (frag, counts)
    assert bench.FP64_INSTR_PER_PAIR == 43


def test_no_cpu_fallback_without_device():
    if N.device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_1301_5914_b200 import (ChargeSystem, PhysicalParams, SolverConfig, discretize,
                                      gmres_solve, icosahedral_sphere)

    with pytest.raises(RuntimeError, match="CUDA device"):
        discretize(icosahedral_sphere(1), PhysicalParams(1, 80, 0.1), ChargeSystem(np.zeros((0, 3)), []),
                   SolverConfig())
    with pytest.raises(RuntimeError, match="CUDA device"):
        gmres_solve(lambda v: v, np.ones(4), SolverConfig())
    from paper_1301_5914_b200 import geometry, kernels

    for call in (lambda: geometry.fit_arc([1, 0, 0], [1, 0, 0], [0, 1, 0], [0, 1, 0]),
                 lambda: geometry.frames_at(np.zeros((1, 10, 3)), np.zeros((1, 10, 3)), [[0.2, 0.2]]),
                 lambda: geometry.nodes_from_vertex_data(*np.eye(3).repeat(2, axis=0)),
                 lambda: kernels.kernel_values_d([1.0, 0, 0], [1.0, 0, 0], [0, 1.0, 0], PhysicalParams(1, 80, 0.1)),
                 lambda: kernels.source_terms([1.0, 0, 0], [1.0, 0, 0], ChargeSystem([[0, 0, 0]], [1.0]))):
        with pytest.raises(RuntimeError, match="CUDA device"):
            call()


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1301_5914_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "hobi_oracle" not in src and "oracle/" not in src, f


def test_public_api_covers_the_reference_surface():
    """Every name in pbbem.__all__ (pkg/src/pbbem/__init__.py:45-73) is importable here."""
    import paper_1301_5914_b200 as P

    reference_all = [
        "ChargeSystem", "DiscretizedProblem", "FlatMesh", "GmresNonConvergence", "PhysicalParams",
        "RunReport", "SolverConfig", "SphereProblem", "SurfaceSolution", "assemble_rhs",
        "convergence_order", "discretize", "gmres_solve", "icosahedral_sphere", "kirkwood_centered",
        "kirkwood_series", "make_operator", "matvec_hobi", "matvec_lobi", "parse_charges",
        "partition_targets", "parse_msms", "radial_project", "solvation_energy", "solve",
        "surface_potential_error", "write_msms"]
    assert [n for n in reference_all if not hasattr(P, n)] == []


def test_header_is_plain_c():
    """include/hobi.h is a C header (no C++ or CUDA types cross the boundary):
    it compiles as strict C99 and a C program can take every entry point."""
    import shutil
    import subprocess
    import tempfile

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    names = _declared()
    src = '#include "hobi.h"\ntypedef void (*fn_t)(void);\nint main(void) {\n  fn_t f;\n'
    src += "".join(f"  f = (fn_t)&{n};\n  (void)f;\n" for n in names if n != "hobi_apply_fn")
    src += "  return 0;\n}\n"
    with tempfile.TemporaryDirectory() as tmp:
        c_file = os.path.join(tmp, "probe.c")
        open(c_file, "w").write(src)
        out = subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-pedantic", "-fsyntax-only",
                              "-I", os.path.join(ROOT, "include"), c_file], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_default_rule_tables_are_generated_from_the_python_rules():
    """csrc/hobi_default_rules.inc (hobi_create_default's tables) is exactly
    what tools/gen_default_rules.py produces from quadrature.py."""
    import subprocess

    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_default_rules.py"), "--check"],
                         capture_output=True, text=True)
    assert out.returncode == 0, "regenerate with python tools/gen_default_rules.py"


def test_c_example_compiles():
    import shutil
    import subprocess
    import tempfile

    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    with tempfile.TemporaryDirectory() as tmp:
        out = subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-pedantic", "-I", os.path.join(ROOT, "include"),
                              os.path.join(ROOT, "examples", "c_solve.c"), "-L", os.path.dirname(N.LIB_PATH),
                              "-lhobi", "-o", os.path.join(tmp, "c_solve")], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_round2_entry_points_validate_arguments_without_a_device():
    """The round-2 C-ABI entries reject bad handles and sizes before they touch
    a device (status codes, no crash), on any machine."""
    import ctypes as C

    import numpy as np

    from paper_1301_5914_b200 import _native as N

    lib = N.load()
    z = np.zeros(4)
    assert lib.hobi_kirkwood_traces(0, N.dptr(z), 1, N.dptr(z), N.dptr(z), 1, N.dptr(z), N.dptr(z), 0,
                                    N.dptr(z), N.dptr(z)) == N.HOBI_ERR_VALUE
    assert lib.hobi_kirkwood_traces(0, N.dptr(z), 0, N.dptr(z), N.dptr(z), 1, N.dptr(z), N.dptr(z), 3,
                                    N.dptr(z), N.dptr(z)) == N.HOBI_OK  # nothing to evaluate
    assert lib.hobi_kirkwood_energy_terms(0, N.dptr(z), N.dptr(z), -1, N.dptr(z), N.dptr(z), 3,
                                          N.dptr(z)) == N.HOBI_ERR_VALUE
    assert lib.hobi_hypot_check(0, N.dptr(z), N.dptr(z), -1, N.dptr(z)) == N.HOBI_ERR_VALUE
    assert lib.hobi_comm_init_p2p(None, 2, 0) == N.HOBI_ERR_STATE
    assert lib.hobi_matvec_p2p_phase(None, N.dptr(z), N.dptr(z), 0) == N.HOBI_ERR_STATE
    assert lib.hobi_group_info(None, None, None, None, None, None) == N.HOBI_ERR_STATE
    ms = np.zeros(1)
    assert lib.hobi_group_bench(None, N.dptr(z), N.dptr(z), 1, 0, 0, N.dptr(ms)) == N.HOBI_ERR_STATE
    assert "null" in N.last_error()
    # the function-level geometry / kernels entries: sizes and null arrays first
    ci = (C.c_int * 1)()
    bad, code = (C.c_int64 * 1)(), (C.c_int * 1)()
    assert lib.hobi_geometry_fit_arcs(0, N.dptr(z), N.dptr(z), N.dptr(z), N.dptr(z), -1, N.dptr(z), ci) == N.HOBI_ERR_VALUE
    assert lib.hobi_geometry_fit_arcs(0, None, N.dptr(z), N.dptr(z), N.dptr(z), 1, N.dptr(z), ci) == N.HOBI_ERR_VALUE
    assert lib.hobi_geometry_arc_normals(0, N.dptr(z), None, N.dptr(z), 1, N.dptr(z), ci) == N.HOBI_ERR_VALUE
    assert lib.hobi_geometry_nodes(0, N.dptr(z), N.dptr(z), 1, N.dptr(z), N.dptr(z), None, code) == N.HOBI_ERR_VALUE
    assert lib.hobi_geometry_nodes(0, None, N.dptr(z), 1, N.dptr(z), N.dptr(z), bad, code) == N.HOBI_ERR_VALUE
    assert lib.hobi_geometry_frames(0, N.dptr(z), N.dptr(z), 1, None, 2, N.dptr(z), N.dptr(z), N.dptr(z), None,
                                    None) == N.HOBI_ERR_VALUE
    assert lib.hobi_geometry_frames(0, N.dptr(z), N.dptr(z), -1, N.dptr(z), 2, N.dptr(z), N.dptr(z), N.dptr(z),
                                    None, None) == N.HOBI_ERR_VALUE
    assert lib.hobi_source_terms(0, N.dptr(z), N.dptr(z), -1, N.dptr(z), N.dptr(z), 1, N.dptr(z),
                                 N.dptr(z)) == N.HOBI_ERR_VALUE
    assert lib.hobi_source_terms(0, N.dptr(z), N.dptr(z), 1, None, N.dptr(z), 1, N.dptr(z),
                                 N.dptr(z)) == N.HOBI_ERR_VALUE
