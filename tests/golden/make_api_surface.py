"""Public names of every pbbem module (top-level classes, functions and
constants without a leading underscore), read from the reference sources in
the build container -> tests/golden/pbbem_api.json.  tests/test_host.py checks
that the same-named module of this package exports each of them."""
import ast
import json
import os
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src/pbbem"
out = {}
for fn in sorted(os.listdir(SRC)):
    if not fn.endswith(".py") or fn.startswith("__"):
        continue
    names = set()
    for node in ast.parse(open(os.path.join(SRC, fn)).read()).body:
        if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
            names.add(node.name)
        elif isinstance(node, ast.Assign):
            names.update(t.id for t in node.targets if isinstance(t, ast.Name))
        elif isinstance(node, ast.AnnAssign) and isinstance(node.target, ast.Name):
            names.add(node.target.id)
    out[fn[:-3]] = sorted(n for n in names if not n.startswith("_"))
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pbbem_api.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1, sort_keys=True)
    fh.write("\n")
print({k: len(v) for k, v in out.items()})
