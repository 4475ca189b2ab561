"""Attribute an ncu --set full capture of k_simulate to engine source functions.

  python tools/ncu_funcs.py <report.ncu-rep> [variant-substring]

Prints, per source function (inlined code attributed by line info), the share
of warp-stall samples, of instruction-fetch (no_instruction) stalls, the
executed SASS footprint and warp instructions executed.  Needs the library
the report was taken with (line info from the cubin) in the working tree.
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
ENGINE = os.path.join(HERE, "paper_2511_21669_b200", "csrc", "device", "engine.cuh")
LIB = os.path.join(HERE, "paper_2511_21669_b200", "libdsdsim.so")


def main(rep, variant="k_simulateILb1ELb0ELb1ELb0ELi2E"):  # (the specialised production kernel)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "stall_no_inst" in r)
    ix = {k: j for j, k in enumerate(rows[hi])}
    data = []
    for r in rows[hi + 1:]:
        try:
            a = int(r[ix["Address"]], 16)
        except (ValueError, IndexError):
            continue
        f = lambda k: float(r[ix[k]] or 0)
        data.append((a, f("Warp Stall Sampling (All Samples)"), f("stall_no_inst"), f("Instructions Executed")))
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
    src = open(ENGINE).read().split("\n")
    fdefs = [(i + 1, l.strip()) for i, l in enumerate(src)
             if re.match(r"\s*(DSD_HD|static DSD_HD|DSD_HD_NOINLINE|static DSD_HD_NOINLINE)\b.*\(", l)]

    def fname(ln):
        if not ln:
            return "?"
        if ln[0] != "engine.cuh":
            return f"{ln[0]}:{ln[1]}"
        name = "?"
        for n, t in fdefs:
            if n <= ln[1]:
                name = t
        return name[:64]

    tot = sum(d[1] for d in data) or 1
    tni = sum(d[2] for d in data) or 1
    tex = sum(d[3] for d in data) or 1
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0, 0.0])
    for a, al, ni, ex in data:
        g = agg[fname(amap.get(a - base))]
        g[0] += al
        g[1] += ni
        g[2] += ex > 0
        g[3] += ex
    print(f"no_instruction share of stalls {100 * tni / tot:.1f}%, executed SASS {sum(d[3] > 0 for d in data)}")
    print(" stall%  fetch%  exec_sz  inst%   function")
    for k, g in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
        print(f"{100 * g[0] / tot:6.1f}  {100 * g[1] / tni:6.1f}  {g[2]:7d}  {100 * g[3] / tex:5.1f}   {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
