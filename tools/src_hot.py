"""Hottest source lines of an ncu source export
(ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv)."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, hdr, fname = [], None, ""
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
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        d = dict(zip(hdr[2:], r[2:]))
        try:
            s = int(r[4]); ni = int(r[5])
        except ValueError:
            continue
        rows.append((s, ni, fname, r[0], r[1][:90], d))
tot = sum(x[0] for x in rows) or 1
print("total samples", tot)
keys = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k] if hdr else []
agg = {k: 0 for k in keys}
for s, ni, fn, ln, src, d in rows:
    for k in keys:
        try:
            agg[k] += int(d.get(k, "0") or 0)
        except ValueError:
            pass
print("stalls:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for s, ni, fn, ln, src, d in sorted(rows, key=lambda x: -x[0])[:top]:
    st = []
    for k in keys:
        try:
            st.append((int(d.get(k, "0") or 0), k[6:]))
        except ValueError:
            pass
    st = " ".join(f"{n}:{100*v/max(s,1):.0f}" for v, n in sorted(st, reverse=True)[:3])
    print(f"{100*s/tot:5.1f}% ni {100*ni/tot:5.1f}%  {fn}:{ln:5s} {src[:70]:70s} [{st}]")
