"""In-tree build of libhobi.so for sm_100a (nvcc -shared; no torch extension).

    python -m paper_1301_5914_b200.build          # build if stale
    python -m paper_1301_5914_b200.build --force  # rebuild

The geometry and literal translation units are compiled with -fmad=false so
their arithmetic rounds exactly like the numpy reference (they write every
fused multiply-add explicitly); the sweep and GMRES units keep contraction on.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libhobi.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", os.path.join(ROOT, "include")]
UNITS = {
    "hobi_api.cu": [],
    "hobi_sweep.cu": [],
    "hobi_gmres.cu": [],
    "hobi_group.cu": [],
    "hobi_msms.cu": [],
    "hobi_geometry.cu": ["-fmad=false"],
    "hobi_literal.cu": ["-fmad=false"],
}
HEADERS = ["hobi_internal.cuh", "hobi_fastmath.cuh", "hobi_default_rules.inc"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in list(UNITS) + HEADERS]
    deps.append(os.path.join(ROOT, "include", "hobi.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    objdir = os.path.join(HERE, "_build")
    os.makedirs(objdir, exist_ok=True)
    objs, cmds = [], []
    for unit, extra in UNITS.items():
        obj = os.path.join(objdir, unit.replace(".cu", ".o"))
        cmd = [nvcc, *ARCH, *COMMON, *extra, "-Xptxas", "-v" if verbose else "-O3", "-c",
               os.path.join(CSRC, unit), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        cmds.append(cmd)
        objs.append(obj)
    # translation units compile independently: run them side by side
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as pool:
        for res in pool.map(lambda c: subprocess.run(c, check=True), cmds):
            del res
    tmp = LIB + ".tmp"
    subprocess.run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"], check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
