"""Per-source-line warp-stall breakdown of an ncu report (development aid).

    python tools/ncu_lines.py <report.ncu-rep> [top]
"""
import csv
import subprocess
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg, fname = {}, None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < len(hdr) or r[0] in ("Line No", ""):
        continue
    agg[(fname, r[0], r[1][:70])] = [f(r[4]), f(r[7])] + [f(r[i]) for i, _ in cols]
tot = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"instructions {ti:.3e}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    st = sorted(((v[2 + j], cols[j][1][6:]) for j in range(len(cols))), reverse=True)[:3]
    print(f"{v[0] / tot * 100:5.1f}% inst {v[1] / ti * 100:5.1f}% {k[0]}:{k[1]} {k[2]}\n        "
          + ", ".join(f"{n} {x / max(v[0], 1) * 100:.0f}%" for x, n in st))
