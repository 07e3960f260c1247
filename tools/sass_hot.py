"""SASS instructions matching a pattern, by executed count, with their CUDA
source line (ncu --page source --csv --print-source cuda,sass export)."""
import csv
import re
import sys

path, pat = sys.argv[1], re.compile(sys.argv[2] if len(sys.argv) > 2 else r"\b(LDL|STL)\b")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
hdr, cur, fname, out = None, "", "", []
with open(path) as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0]:
            cur = f"{fname}:{r[0]} {r[1].strip()[:60]}"
            continue
        if len(r) > 7 and pat.search(r[3]):
            try:
                n = int(r[7])
            except ValueError:
                continue
            out.append((n, int(r[4] or 0), r[3].strip()[:50], cur))
tot = sum(x[0] for x in out)
print("matching instructions executed:", tot)
for n, s, ins, src in sorted(out, reverse=True)[:top]:
    print(f"{n:12d} samp {s:6d}  {ins:50s} {src}")
