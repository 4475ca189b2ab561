"""Summarise ncu captures into profiles/ (tracked).

  python tools/ncu_summary.py full  <report.ncu-rep> <out.json>   # --set full capture of k_simulate
  python tools/ncu_summary.py launches <launches.csv> <out.json>  # gpu__time_duration launch list

The full-capture summary keeps what the roofline and DESIGN.md cite: kernel
time, DRAM bytes (the bench's `roofline.traffic`), cache hit rates, issue and
occupancy figures, warp-stall breakdown and the hottest source lines.
"""
import collections
import csv
import io
import json
import subprocess
import sys


TIME_TO_MS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
              "second": 1e3}


def ncu_csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep, out_path):
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, vals = rows[0], rows[2]
    d = dict(zip(hdr, vals))

    def f(k):
        try:
            return float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return None

    stalls = {}
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v)
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    stall_pct = {k: round(100 * v / tot, 2) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v > 0}
    dram_r = f("dram__bytes_read.sum")
    dram_w = f("dram__bytes_write.sum")
    units = dict(zip(hdr, rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def bytes_of(k):
        v = f(k)
        return None if v is None else v * scale.get(units.get(k, "byte"), 1)

    summary = {
        "kernel": d.get("Kernel Name"),
        "grid": d.get("Grid Size"), "block": d.get("Block Size"),
        "duration_ms_under_ncu": (f("gpu__time_duration.sum") or 0) * TIME_TO_MS.get(units.get("gpu__time_duration.sum"), 1.0),
        "dram_bytes_read": bytes_of("dram__bytes_read.sum"),
        "dram_bytes_write": bytes_of("dram__bytes_write.sum"),
        "dram_bytes_per_launch": (bytes_of("dram__bytes_read.sum") or 0) + (bytes_of("dram__bytes_write.sum") or 0),
        "dram_throughput_pct_of_peak": f("dram__bytes_read.sum.pct_of_peak_sustained_elapsed"),
        "l1_hit_pct": f("l1tex__t_sector_hit_rate.pct"),
        "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": f("smsp__inst_executed.sum"),
        "threads_per_instruction": f("smsp__thread_inst_executed_per_inst_executed.ratio"),
        "registers_per_thread": f("launch__registers_per_thread"),
        "stall_pct": stall_pct,
    }
    # hottest source lines by stall samples
    src = ncu_csv(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"])
    lines = collections.defaultdict(lambda: [0.0, ""])
    cur = None
    for r in src:
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0].isdigit():
            try:
                lines[(cur, int(r[0]))][0] += float(r[4] or 0)
                lines[(cur, int(r[0]))][1] = r[1].strip()[:100]
            except (ValueError, IndexError):
                pass
    t = sum(v[0] for v in lines.values()) or 1.0
    summary["hot_lines"] = [
        {"file": k[0], "line": k[1], "stall_pct": round(100 * v[0] / t, 2), "source": v[1]}
        for k, v in sorted(lines.items(), key=lambda x: -x[1][0])[:20]]
    with open(out_path, "w") as fo:
        json.dump(summary, fo, indent=1)
    print(json.dumps({k: summary[k] for k in ("kernel", "dram_bytes_per_launch", "l1_hit_pct", "l2_hit_pct",
                                              "issue_active_pct", "threads_per_instruction")}))


def launches(csv_path, out_path):
    rows = [r for r in csv.reader(open(csv_path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ix = {k: i for i, k in enumerate(hdr)}
    per = collections.defaultdict(list)
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        per[name].append(v * TIME_TO_MS.get(unit, 1.0))
    tot = sum(sum(v) for v in per.values()) or 1.0
    summary = {k: {"launches": len(v), "total_ms": round(sum(v), 3), "share_pct": round(100 * sum(v) / tot, 2)}
               for k, v in sorted(per.items(), key=lambda x: -sum(x[1]))}
    with open(out_path, "w") as fo:
        json.dump(summary, fo, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
