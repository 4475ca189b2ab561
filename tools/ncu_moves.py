"""Executed register moves (IMAD.MOV / MOV) of one kernel per source line,
from an ncu --set full capture (see ncu_funcs.py); with --all, every executed
instruction per source line; with --stall=<reason> (long_sb, wait, ...), that
reason's warp-stall samples per source line.

  python tools/ncu_moves.py <report.ncu-rep> [kernel-substring] [--all | --stall=long_sb]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEV = os.path.join(HERE, "paper_2511_21669_b200", "csrc", "device")
LIB = os.path.join(HERE, "paper_2511_21669_b200", "libdsdsim.so")


def main(rep, variant="k_simulateILb1ELb0ELb1ELb0", *flags):
    every = "--all" in flags
    stall = next((f.split("=", 1)[1] for f in flags if f.startswith("--stall=")), None)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    ix = {k: j for j, k in enumerate(rows[hi])}
    data = []
    for r in rows[hi + 1:]:
        try:
            a = int(r[ix["Address"]], 16)
            ex = float(r[ix["stall_" + stall if stall else "Instructions Executed"]] or 0)
        except (ValueError, IndexError):
            continue
        t = r[ix["Source"]].split()
        op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?"))
        data.append((a, op, ex))
    base = min(d[0] for d in data)
    with tempfile.TemporaryDirectory() as td:
        subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=td, check=True, capture_output=True)
        cub = [x for x in os.listdir(td) if x.startswith("runtime")][0]
        dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(td, cub)], capture_output=True,
                             text=True).stdout
    amap, fn, line = {}, None, None
    for l in dis.split("\n"):
        m = re.search(r"^\s*\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
        m = re.search(r'## File "([^"]+)", line (\d+)', l)
        if m:
            line = (os.path.basename(m.group(1)), int(m.group(2)))
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", l)
        if m and fn and variant in fn:
            amap[int(m.group(1), 16)] = line
    srcs = {}
    tot = sum(d[2] for d in data) or 1
    mv = collections.Counter()
    allc = collections.Counter()
    for a, op, ex in data:
        ln = amap.get(a - base)
        allc[ln] += ex
        if every or stall or op.startswith("IMAD.MOV") or op == "MOV" or op.startswith("MOV."):
            mv[ln] += ex
    tm = sum(mv.values())
    what = f"stall_{stall} samples" if stall else ("all" if every else "moves")
    print(f"{what}: {100 * tm / tot:.1f}% (of the column total)")
    for ln, ex in mv.most_common(30):
        text = ""
        if ln:
            f = os.path.join(DEV, ln[0])
            if os.path.exists(f):
                srcs.setdefault(f, open(f).read().split("\n"))
                text = srcs[f][ln[1] - 1].strip()[:90]
        print(f"{100 * ex / tot:5.2f}%  (line total {100 * allc[ln] / tot:5.2f}%)  {ln}  {text}")


if __name__ == "__main__":
    main(*sys.argv[1:])
