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
    "hobi_singular.cu": [],
    "hobi_gmres.cu": [],
    "hobi_group.cu": [],
    "hobi_msms.cu": [],
    "hobi_geometry.cu": ["-fmad=false"],
    "hobi_literal.cu": ["-fmad=false"],
    "hobi_kirkwood.cu": ["-fmad=false"],
}
HEADERS = ["hobi_internal.cuh", "hobi_fastmath.cuh", "hobi_tma.cuh", "hobi_default_rules.inc"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def _deps():
    deps = [os.path.join(CSRC, f) for f in list(UNITS) + HEADERS]
    deps.append(os.path.join(ROOT, "include", "hobi.h"))
    deps.append(os.path.abspath(__file__))
    return deps


def source_hash() -> str:
    """SHA-256 over the library's sources and this recipe (content, not
    mtimes: a repo snapshot copied to another machine keeps its built library)."""
    import hashlib

    h = hashlib.sha256()
    for d in _deps():
        with open(d, "rb") as f:
            h.update(os.path.basename(d).encode() + b"\0" + f.read())
    return h.hexdigest()


STAMP = LIB + ".srchash"


def _stale():
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


def sources_present() -> bool:
    """False on a box that received only the built library."""
    return all(os.path.exists(os.path.join(CSRC, f)) for f in UNITS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    stamp = source_hash()  # of the sources this build compiles
    # objects and the temporary library are private to this process, so two
    # builders can never interleave writes into one file
    objdir = os.path.join(HERE, "_build", f"p{os.getpid()}")
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
    tmp = f"{LIB}.{os.getpid()}.tmp"
    subprocess.run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"], check=True)
    os.replace(tmp, LIB)
    with open(STAMP + ".tmp", "w") as f:
        f.write(stamp + "\n")
    os.replace(STAMP + ".tmp", STAMP)
    import shutil

    shutil.rmtree(objdir, ignore_errors=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
