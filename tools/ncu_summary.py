"""Summarise ncu output (launch-list CSV and/or a --set full report) into a
small markdown file for profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --report gpurun_out/prof_c2.ncu-rep --out profiles/r01_c2.md --title "..."
"""
import argparse
import csv
import io
import statistics
import subprocess
from collections import OrderedDict, defaultdict

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "SM Frequency"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("Memory Workload Analysis", "Memory Throughput"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Scheduler Statistics", "No Eligible"),
    ("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Occupancy", "Achieved Occupancy"),
    ("Occupancy", "Theoretical Occupancy"),
]


def short(name):
    name = name.replace("void ", "").replace("dopt::", "")
    return name.split("(")[0][:70]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = OrderedDict()
    for r in rows[hi + 1:]:
        per.setdefault(r[0], {"name": short(r[ki])})[r[mi]] = float(r[vi].replace(",", ""))
    agg = defaultdict(list)
    for d in per.values():
        agg[d["name"]].append(d)
    out = ["| kernel | launches | median time (us) | DRAM read MB | DRAM write MB | share of time |",
           "|---|---|---|---|---|---|"]
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())
    for name, ds in agg.items():
        t = [d.get("gpu__time_duration.sum", 0) / 1e3 for d in ds]
        rd = [d.get("dram__bytes_read.sum", 0) / 1e6 for d in ds]
        wr = [d.get("dram__bytes_write.sum", 0) / 1e6 for d in ds]
        share = sum(d.get("gpu__time_duration.sum", 0) for d in ds) / tot if tot else 0
        out.append(f"| `{name}` | {len(ds)} | {statistics.median(t):.2f} | "
                   f"{statistics.median(rd) if rd else 0:.1f} | {statistics.median(wr) if wr else 0:.1f} | "
                   f"{share:.1%} |")
    return "\n".join(out)


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    kernels = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = (d["ID"], short(d["Kernel Name"]))
        kernels.setdefault(k, {})[(d["Section Name"], d["Metric Name"])] = (d["Metric Value"], d["Metric Unit"])
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rawd = {}
    if len(rr) > 2:
        hh = rr[0]
        for r in rr[2:]:
            d = dict(zip(hh, r))
            rawd[d.get("ID")] = d
    out = []
    for (kid, name), m in kernels.items():
        out.append(f"### `{name}` (ID {kid})\n")
        out.append("| metric | value |\n|---|---|")
        for key in KEYS:
            if key in m:
                v, u = m[key]
                out.append(f"| {key[1]} | {v} {u} |")
        d = rawd.get(kid, {})
        for met in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if met in d:
                out.append(f"| {met} | {d[met]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    parts = [f"# {a.title}\n", a.note + "\n" if a.note else ""]
    if a.launches:
        parts += ["## Launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                  "dram__bytes_write.sum --clock-control none; cold-cache, serialised)\n",
                  launches(a.launches), ""]
    if a.report:
        parts += ["## ncu --set full (top kernels)\n", report(a.report)]
    open(a.out, "w").write("\n".join(parts))
    print(a.out)
