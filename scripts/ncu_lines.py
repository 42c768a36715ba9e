"""Per-source-line warp-stall samples of an ncu report (--print-source cuda,sass;
dev aid): python scripts/ncu_lines.py REPORT [TOP]"""
import csv, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, line, src = None, None, {}
samples = defaultdict(float)
ls = defaultdict(float)
hdr = None
for row in csv.reader(out.splitlines()):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].rsplit("/", 1)[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or row[0] == "Function Name":
        continue
    if row[0]:  # a source line row
        line = (fname, int(row[0]))
        src[line] = row[1].strip()
        continue
    # sass row under the current source line
    try:
        s = float(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    samples[line] += s
tot = sum(samples.values()) or 1
for k, v in sorted(samples.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * v / tot:5.1f}%  {k[0]}:{k[1]:<5d} {src.get(k, '')[:110]}")
