"""Summarise ncu outputs for profiles/: a launch-list CSV (gpu__time_duration
per launch) into per-kernel totals/shares, and an ncu-rep (--set full) into the
key per-kernel metrics. Usage:
    python tools/ncu_summary.py launches <launches.csv> [first_id last_id]
    python tools/ncu_summary.py report <prof.ncu-rep>
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, lo=None, hi=None):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    if lo is not None:
        data = [d for d in data if lo <= int(d["ID"]) <= hi]
    tot = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        if "cub::" in name:
            name = "cub::" + name.split("::")[-1].split("<")[0]
        t = float(d["Metric Value"]) / 1e3  # ns -> us
        tot.setdefault(name, [0, 0.0])
        tot[name][0] += 1
        tot[name][1] += t
    s = sum(v[1] for v in tot.values())
    print(f"| kernel | launches | device us (ncu, serialised, cold) | share |")
    print("|---|---|---|---|")
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {n} | {t:.1f} | {100 * t / s:.1f}% |")
    print(f"| **total** | {sum(v[0] for v in tot.values())} | {s:.1f} | 100% |")


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Issue Slots Busy", "Executed Instructions", "Achieved Occupancy", "Registers Per Thread",
        "No Eligible", "Avg. Active Threads Per Warp", "Warp Cycles Per Issued Instruction"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    idx = {n: i for i, n in enumerate(h)}
    per = collections.OrderedDict()
    for row in r[1:]:
        m = row[idx["Metric Name"]]
        if m in WANT:
            key = (row[idx["ID"]], row[idx["Kernel Name"]].split("(")[0].replace("void ", ""))
            per.setdefault(key, {})[m] = f'{row[idx["Metric Value"]]} {row[idx["Metric Unit"]]}'.strip()
    for (i, k), ms in per.items():
        print(f"### {k} (launch {i})")
        for m in WANT:
            if m in ms:
                print(f"- {m}: {ms[m]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if rr:
        h = rr[0]
        cols = [i for i, n in enumerate(h) if n in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
        ki = h.index("Kernel Name") if "Kernel Name" in h else None
        print("\n| kernel | dram__bytes_read.sum | dram__bytes_write.sum |")
        print("|---|---|---|")
        for row in rr[2:]:
            if ki is not None and cols:
                print(f"| {row[ki].split('(')[0]} | " + " | ".join(f"{row[c]} {rr[1][c]}" for c in cols) + " |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        a = sys.argv[2:]
        launches(a[0], int(a[1]) if len(a) > 1 else None, int(a[2]) if len(a) > 2 else None)
    else:
        report(sys.argv[2])
