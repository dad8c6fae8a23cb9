"""Drop-in check: run the reference package's OWN test files, unmodified,
against this repo's package (every `pbbem` import aliased to
`paper_1301_5914_b200` by the pbbem_alias pytest plugin) on a GPU box.

The reference's tests are not part of this repo.  `--stage` copies them from
/root/reference/pkg/tests (build container only) into baseline/_ref/tests_pbbem/,
which is git-ignored like the reference install next to it but travels to the
GPU box with the snapshot; the run itself reads only that staged copy.

    python tests/checks/reference_suite.py --stage          # build container
    gpurun -- python tests/checks/reference_suite.py        # GPU box
    python tests/checks/reference_suite.py -- -k kirkwood   # extra pytest args after --
    python tests/checks/reference_suite.py --scripts        # the reference's scripts/ instead of its tests

Prints pytest's per-file counts and one JSON summary line; exit code = pytest's.
"""

from __future__ import annotations

import json
import os
import re
import shutil
import stat
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
STAGED = os.path.join(ROOT, "baseline", "_ref", "tests_pbbem")
SOURCE = "/root/reference/pkg/tests"
STAGED_SCRIPTS = os.path.join(ROOT, "baseline", "_ref", "scripts_pbbem")
SOURCE_SCRIPTS = "/root/reference/pkg/scripts"
# reference scripts (unmodified) and the arguments of the runs recorded in profiles/r02_reference_suite.md
SCRIPT_RUNS = (("sphere_convergence.py", ["--levels", "1", "2", "3"]),
               ("sphere_convergence.py", ["--eccentric", "--levels", "2", "3", "4"]),
               ("worker_scaling.py", ["--level", "2", "--workers", "1", "2", "4"]))


def stage() -> int:
    if not os.path.isdir(SOURCE):
        print(f"{SOURCE} not found (staging runs in the build container)", file=sys.stderr)
        return 2
    shutil.rmtree(STAGED, ignore_errors=True)
    shutil.copytree(SOURCE, STAGED, ignore=shutil.ignore_patterns("__pycache__", ".hypothesis"))
    print(f"staged {len(os.listdir(STAGED))} files into {os.path.relpath(STAGED, ROOT)}")
    shutil.rmtree(STAGED_SCRIPTS, ignore_errors=True)
    shutil.copytree(SOURCE_SCRIPTS, STAGED_SCRIPTS, ignore=shutil.ignore_patterns("__pycache__"))
    print(f"staged {len(os.listdir(STAGED_SCRIPTS))} files into {os.path.relpath(STAGED_SCRIPTS, ROOT)}")
    return 0


def run_scripts() -> int:
    """The reference's scripts/, files untouched, with pbbem aliased to this package."""
    if not os.path.isdir(STAGED_SCRIPTS):
        print(f"{STAGED_SCRIPTS} missing: run with --stage in the build container first", file=sys.stderr)
        return 2
    env = dict(os.environ)
    env["PYTHONPATH"] = HERE + os.pathsep + ROOT + os.pathsep + env.get("PYTHONPATH", "")
    worst = 0
    for name, argv in SCRIPT_RUNS:
        path = os.path.join(STAGED_SCRIPTS, name)
        code = ("import sys, runpy, warnings; warnings.simplefilter('ignore'); import pbbem_alias; "
                f"sys.argv = {[path] + argv!r}; runpy.run_path({path!r}, run_name='__main__')")
        print(f"$ {name} {' '.join(argv)}", flush=True)
        proc = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(proc.stdout + proc.stderr[-3000:], flush=True)
        worst = max(worst, proc.returncode)
    return worst


def main(argv) -> int:
    if "--stage" in argv:
        return stage()
    if "--scripts" in argv:
        return run_scripts()
    extra = argv[argv.index("--") + 1:] if "--" in argv else []
    if not os.path.isdir(STAGED):
        print(f"{STAGED} missing: run with --stage in the build container first", file=sys.stderr)
        return 2
    with tempfile.TemporaryDirectory() as tmp:
        # the one subprocess test looks for the console script on PATH (ref tests/test_cli.py:309)
        exe = os.path.join(tmp, "pbbem")
        with open(exe, "w") as f:
            f.write(f'#!/bin/sh\nPYTHONPATH="{ROOT}" exec "{sys.executable}" -m paper_1301_5914_b200 "$@"\n')
        os.chmod(exe, os.stat(exe).st_mode | stat.S_IEXEC)
        env = dict(os.environ)
        env["PATH"] = tmp + os.pathsep + env.get("PATH", "")
        env["PYTHONPATH"] = HERE + os.pathsep + ROOT + os.pathsep + env.get("PYTHONPATH", "")
        cmd = [sys.executable, "-m", "pytest", "-p", "pbbem_alias", STAGED, "-q", "--no-header", "-p",
               "no:cacheprovider", "-rf", "--rootdir", STAGED] + extra
        proc = subprocess.run(cmd, env=env, cwd=tmp, capture_output=True, text=True)
    out = proc.stdout + proc.stderr
    print(out[-12000:])
    tail = [ln for ln in out.splitlines() if re.search(r"\d+ (passed|failed|error)", ln)]
    counts = {k: int(v) for v, k in re.findall(r"(\d+) (passed|failed|errors?|skipped|xfailed|deselected)",
                                               tail[-1] if tail else "")}
    print(json.dumps({"reference_suite": counts, "rc": proc.returncode}))
    return proc.returncode


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
