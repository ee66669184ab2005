"""Print the key fields of bench.py JSON lines and per-launch ncu times:
    python tools/bsum.py bench <log>...      python tools/bsum.py launches <csv> [lo hi]"""
import csv
import json
import sys


def bench(paths):
    for p in paths:
        for l in open(p):
            if l.startswith("{"):
                d = json.loads(l)
                print(p, "val %.1f G" % (d["value"] / 1e9), "ms %.3f" % d["ms_per_step"],
                      {k: round(v, 3) for k, v in d.get("phases_ms", {}).items()},
                      "frac %.3f" % d["roofline"]["frac"], "e2e %.2f G" % (d["e2e"]["value"] / 1e9),
                      "launches", d.get("gpu_launches"),
                      "labelled %.1f G" % (d["extra"]["labelled"]["points_per_s"] / 1e9) if "extra" in d else "")
            elif "rror" in l:
                print(p, l.strip())


def launches(path, lo=0, hi=10**9):
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if lo <= int(d["ID"]) <= hi:
                print(d["ID"], d["Kernel Name"][:60], d["Metric Value"])


if __name__ == "__main__":
    if sys.argv[1] == "bench":
        bench(sys.argv[2:])
    else:
        a = sys.argv[2:]
        launches(a[0], *(int(v) for v in a[1:]))
