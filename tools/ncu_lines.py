"""Rank CUDA source lines of one kernel in an ncu report by warp-stall samples:
    python tools/ncu_lines.py <rep> <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
ix = {n: i for i, n in enumerate(hdr)}
si, ki = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
ti = ix.get("Avg. Threads Executed")


def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


lines = [r for r in rows if len(r) == len(hdr) and r[0] not in ("", hdr[0])]
tot = sum(f(r[si]) for r in lines)
print(f"total stall samples {tot:.0f}, warp instructions {sum(f(r[ki]) for r in lines) / 1e6:.1f}M")
for r in sorted(lines, key=lambda r: -f(r[si]))[:top]:
    print(f"{100 * f(r[si]) / tot:5.1f}% {f(r[ki]) / 1e6:7.2f}M thr={r[ti] if ti else '-':>4} L{r[0]}: {r[1].strip()[:90]}")
