"""Summarise a gpurun_out/<tag>/ directory into profiles/<round>/ (tracked).

  python tools/summarize_profiles.py gpurun_out/r01a profiles/r01

Writes:
  launches_step.csv   per-kernel share of the LAST decode step in the ncu launch
                      list (gpu__time_duration.sum, cold-cache, serialised)
  ncu_<name>.csv      selected counters of each full-set capture (*.ncu-rep)
  bench.json          the bench line of that call
"""
import collections
import csv
import glob
import io
import os
import shutil
import subprocess
import sys

COUNTERS = [
    "Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def launches(src, dst, per_step):
    rows = list(csv.reader(open(src)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    tail = data[-per_step:] if per_step else data
    agg = collections.OrderedDict()
    for d in tail:
        k = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    with open(dst, "w") as f:
        f.write("kernel,launches,total_us,share,us_per_launch\n")
        for k, (n, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"\"{k}\",{n},{s / 1e3:.2f},{s / tot:.4f},{s / n / 1e3:.2f}\n")
        f.write(f"TOTAL,{sum(v[0] for v in agg.values())},{tot / 1e3:.2f},1.0,\n")
    return tot


def ncu_summary(rep, dst):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if not rows:
        return
    hdr = rows[0]
    idx = [(c, hdr.index(c)) for c in COUNTERS if c in hdr]
    with open(dst, "w") as f:
        f.write(",".join(c for c, _ in idx) + "\n")
        for r in rows[2:]:
            f.write(",".join("\"" + r[i].replace("\"", "") + "\"" for _, i in idx) + "\n")


def main():
    src, dst = sys.argv[1], sys.argv[2]
    per_step = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    os.makedirs(dst, exist_ok=True)
    if os.path.exists(os.path.join(src, "launches.csv")):
        launches(os.path.join(src, "launches.csv"), os.path.join(dst, "launches_step.csv"), per_step)
    for rep in glob.glob(os.path.join(src, "*.ncu-rep")):
        name = os.path.splitext(os.path.basename(rep))[0]
        ncu_summary(rep, os.path.join(dst, f"ncu_{name}.csv"))
    for f in ("bench.json", "pytest_gpu.log", "smoke.log"):
        if os.path.exists(os.path.join(src, f)):
            shutil.copy(os.path.join(src, f), os.path.join(dst, f))


if __name__ == "__main__":
    main()
