"""Summarises ncu captures for profiles/.

    python tools/ncu_summary.py <report.ncu-rep> <out-prefix> [workload]
        writes <out-prefix>.txt (human) and merges per-kernel DRAM bytes per
        launch into profiles/ncu_summary.json (read by bench.py for `traffic`)
        under "<kernel>@<workload>" (and the plain "<kernel>" for the
        headline workload lircmop13-1m)
    python tools/ncu_summary.py --launches <launches.csv> <out.txt>
        condenses a `--metrics gpu__time_duration.sum` launch list into
        per-kernel counts, mean time and share of the profiled span
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

TIME_US = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration_us", 1e-3),
    ("dram__bytes_read.sum", "dram_read_MB", 1.0),
    ("dram__bytes_write.sum", "dram_write_MB", 1.0),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1.0),
    ("smsp__inst_executed.sum", "warp_instructions", 1.0),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct", 1.0),
    ("launch__registers_per_thread", "registers", 1.0),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct", 1.0),
]


def short(name):
    m = re.search(r"(vary_eval_kernel<[^>]*>|\w+_kernel)", name)
    return m.group(1) if m else name[:40]


def kernel_key(name):
    for k in ("vary_eval", "select", "op1", "end_gen", "restore"):
        if k in name:
            return k
    return short(name)


def units_of(raw_hdr, raw_units):
    return dict(zip(raw_hdr, raw_units))


def summarize(rep, prefix, workload="lircmop13-1m"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    u = units_of(hdr, units)
    lines, js = [], {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        rec = {}
        for key, label, scale in METRICS:
            v = d.get(key)
            if v in (None, ""):
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            unit = u.get(key, "")
            if label.endswith("_MB"):
                x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "B": 1e-6, "KB": 1e-3,
                         "MB": 1.0, "GB": 1e3}.get(unit, 1.0)
            if label == "duration_us":
                x = x * TIME_US.get(unit, 1.0)
            rec[label] = round(x, 4)
        lines.append(f"{short(name)}: " + ", ".join(f"{k}={v}" for k, v in rec.items()))
        k = kernel_key(name)
        if "dram_read_MB" in rec and "dram_write_MB" in rec:
            e = {"dram_bytes_per_launch": (rec["dram_read_MB"] + rec["dram_write_MB"]) * 1e6,
                 "source": os.path.basename(rep), **rec}
            js[f"{k}@{workload}"] = e
            if workload == "lircmop13-1m":
                js[k] = e
    with open(prefix + ".txt", "w") as f:
        f.write(f"ncu --set full capture: {os.path.basename(rep)}\n" + "\n".join(lines) + "\n")
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    cur = {}
    if os.path.exists(path):
        with open(path) as f:
            cur = json.load(f)
    cur.update(js)
    with open(path, "w") as f:
        json.dump(cur, f, indent=1, sort_keys=True)
    print("\n".join(lines))


def launches(csv_path, out_txt):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if len(r) != len(hdr) or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v *= TIME_US.get(r[ui], 1.0)
        agg[short(r[ki])].append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"launch list {os.path.basename(csv_path)}: {sum(len(v) for v in agg.values())} launches, "
             f"{tot:.1f} us total (ncu: cold-cache, serialised — compare shares)"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"  {k:45s} n={len(v):4d} mean={sum(v) / len(v):9.2f} us share={sum(v) / tot * 100:5.1f}%")
    open(out_txt, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        summarize(sys.argv[1], sys.argv[2], *sys.argv[3:4])
