"""Summarise a ptxas -v log: registers / spills per solve_kernel instantiation."""
import re
import subprocess
import sys

log = open(sys.argv[1]).read().split("\n")
cur = None
for line in log:
    m = re.search(r"Compiling entry function '(\w+)'", line) or re.search(r"Function properties for (\w+)", line)
    if m:
        cur = m.group(1)
    if cur and "solve_kernel" in cur and ("spill" in line or "registers" in line):
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        name = name.replace("hcb::solve::", "").replace("void solve_kernel", "")
        print(f"{name[:90]:90s} {line.strip()[:80]}")
