"""Executed warp instructions per CUDA source line and per SASS opcode class
from an ncu source export (--page source --csv --print-source cuda,sass)."""
import collections
import csv
import re
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, line, src = "", None, ""
per_line = collections.Counter()
text = {}
per_op = collections.Counter()
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:  # a source line row
        line = (fname, r[0])
        text[line] = r[1].strip()[:80]
        continue
    if len(r) > 7 and r[3] not in ("...", "-"):
        try:
            n = int(r[7])
        except ValueError:
            continue
        per_line[line] += n
        op = re.sub(r"^@!?U?P\w+\s+", "", r[3].strip()).split()[0] if r[3].strip() else "?"
        per_op[op.split(".")[0]] += n
tot = sum(per_line.values()) or 1
print(f"total warp instructions {tot:.3e}")
print("by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in per_op.most_common(22)))
for (f, ln), n in per_line.most_common(top):
    print(f"{100 * n / tot:5.1f}%  {f}:{ln:5s} {text.get((f, ln), '')}")
