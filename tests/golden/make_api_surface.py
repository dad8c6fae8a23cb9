"""Public names of every pbbem module (top-level classes, functions and
constants without a leading underscore), read from the reference sources in
the build container -> tests/golden/pbbem_api.json.  tests/test_host.py checks
that the same-named module of this package exports each of them, that every
public function takes the same positional parameters in the same order, and
that every dataclass carries the same fields."""
import ast
import json
import os
import sys

SRC = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src/pbbem"
out, sigs, fields = {}, {}, {}
for fn in sorted(os.listdir(SRC)):
    if not fn.endswith(".py") or fn.startswith("__"):
        continue
    names = set()
    for node in ast.parse(open(os.path.join(SRC, fn)).read()).body:
        if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
            names.add(node.name)
            if node.name.startswith("_"):
                continue
            if isinstance(node, ast.FunctionDef):  # positional parameter names, in order
                sigs.setdefault(fn[:-3], {})[node.name] = [a.arg for a in node.args.posonlyargs + node.args.args]
            else:  # annotated class attributes = dataclass fields, in order
                attrs = [n.target.id for n in node.body
                         if isinstance(n, ast.AnnAssign) and isinstance(n.target, ast.Name)]
                if attrs:
                    fields.setdefault(fn[:-3], {})[node.name] = attrs
        elif isinstance(node, ast.Assign):
            names.update(t.id for t in node.targets if isinstance(t, ast.Name))
        elif isinstance(node, ast.AnnAssign) and isinstance(node.target, ast.Name):
            names.add(node.target.id)
    out[fn[:-3]] = sorted(n for n in names if not n.startswith("_"))
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pbbem_api.json")
with open(path, "w") as fh:
    json.dump({"names": out, "signatures": sigs, "fields": fields}, fh, indent=1, sort_keys=True)
    fh.write("\n")
print({k: len(v) for k, v in out.items()})
