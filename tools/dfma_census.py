"""Static SASS census of the default sweep kernel's FP64 instructions: how many
DFMAs read three distinct register pairs with no reuse-cache operand (the
pattern that issues at 2/3 of the FP64 rate on B200, profiles/README.md).

    python tools/dfma_census.py [path/to/libhobi.so]
"""
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1301_5914_b200/libhobi.so"
KERNEL = "sweep_kernelILi1ELb1ELb0ELi7ELi2ELi3ELb1E"  # <kScreened, FULL, !SELF, R=7, MINB=2, UNROLL=3, STEP>

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
body, on = [], False
for line in sass.splitlines():
    if "Function :" in line:
        on = KERNEL in line
        continue
    if on:
        body.append(line)
ops = {"DFMA": 0, "DMUL": 0, "DADD": 0}
three = plain3 = 0
for line in body:
    m = re.search(r"\b(DFMA|DMUL|DADD)\b", line)
    if not m:
        continue
    ops[m.group(1)] += 1
    if m.group(1) != "DFMA":
        continue
    f = re.search(r"DFMA(\.\w+)*\s+R\d+,\s*([^,]+),\s*([^,]+),\s*([^;]+);", line)
    operands = [f.group(i).strip() for i in (2, 3, 4)]
    regs = [re.sub(r"[-|]", "", o).split(".")[0] for o in operands if re.match(r"-?\|?R\d", o)]
    if len(regs) == 3 and len(set(regs)) == 3:
        three += 1
        plain3 += not any(".reuse" in o for o in operands)
print(f"{KERNEL}: {ops}, DFMA with 3 distinct registers {three}, of which no reuse operand {plain3}")
