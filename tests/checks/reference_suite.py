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


def stage() -> int:
    if not os.path.isdir(SOURCE):
        print(f"{SOURCE} not found (staging runs in the build container)", file=sys.stderr)
        return 2
    shutil.rmtree(STAGED, ignore_errors=True)
    shutil.copytree(SOURCE, STAGED, ignore=shutil.ignore_patterns("__pycache__", ".hypothesis"))
    print(f"staged {len(os.listdir(STAGED))} files into {os.path.relpath(STAGED, ROOT)}")
    return 0


def main(argv) -> int:
    if "--stage" in argv:
        return stage()
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
