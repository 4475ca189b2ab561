"""Top source lines of an ncu source-page export (--print-source cuda,sass --csv).
  python tools/scratch/src_hot.py <export.csv> [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur, hdr, lines = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif r and r[0].isdigit() and hdr:
        d = dict(zip(hdr, r))
        num = lambda x: int(x) if x.strip().lstrip("-").isdigit() else 0
        lines.append((num(d["# Samples"]), num(d["Instructions Executed"]), cur, r[0], r[1][:90]))
ts = sum(x[0] for x in lines)
ti = sum(x[1] for x in lines)
print("samples", ts, "instructions", ti)
for s, i, f, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{100*s/ts:5.1f}% {100*i/ti:5.1f}%i {f}:{ln} {src}")
