"""SASS rows attributed to one CUDA source line (by line number), with samples."""
import csv, sys
path, line = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
hdr=None; cur=None; rows=[]
for r in csv.reader(open(path)):
    if not r: continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] in ("File Path", "Function Name"): continue
    if r[0]: cur = r[0]; continue
    if cur == line and len(r) > 7:
        try: rows.append((int(r[4] or 0), int(r[7] or 0), r[2], r[3].strip()))
        except ValueError: pass
print(len(rows), "sass rows; total samples", sum(x[0] for x in rows), "executed", sum(x[1] for x in rows))
for s, n, a, ins in sorted(rows, reverse=True)[:top]:
    print(f"{s:7d} {n:12d} {a} {ins[:70]}")
