"""Per-instruction warp-stall breakdown of one kernel from an .ncu-rep (source page, SASS):
    python tools/ncu_stalls.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kre:
    cmd += ["-k", f"regex:{kre}", "-c", "1"]
rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = {k: 0 for k in reasons}
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        n = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        rs = {k: int(r[idx[k]] or 0) for k in reasons}
    except ValueError:  # a repeated header (several kernels in one report)
        continue
    for k in reasons:
        tot[k] += rs[k]
    data.append((n, r[idx["Address"]][-5:], r[idx["Source"]].strip(), r[idx["Instructions Executed"]], rs))
T = sum(d[0] for d in data) or 1
print("samples", T, "by reason:", {k[6:]: round(v / T * 100, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
for n, a, src, ex, rs in sorted(data, key=lambda x: -x[0])[:top]:
    main = sorted(rs.items(), key=lambda x: -x[1])[:2]
    print(f"{n / T * 100:5.1f}% {a} x{ex:>7} {src[:70]:70s} {[(k[6:], v) for k, v in main if v]}")
