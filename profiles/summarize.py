"""Summarize ncu outputs for profiles/ (run here, on the CPU box):
    python profiles/summarize.py <launches.csv> [<prof.ncu-rep> [<traffic.json> <config>]] > profiles/<name>.md
Launch list: per-kernel count, device time and share of the profiled solve
(cold-cache, serialised: shares matter, not absolutes).  Full capture: per
launch duration, DRAM bytes read+write, DRAM throughput % and occupancy."""
import collections
import csv
import os
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        v = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"## Launch list ({sum(v[0] for v in agg.values())} launches, {tot/1e3:.3f} ms total device time)\n")
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k[:70]}` | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% |")
    print()


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_shared_mem"]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    print("## Full-set capture (per launch)\n")
    print("| kernel | time | DRAM read | DRAM write | DRAM % of peak | warps active % | regs | grid |")
    print("|---|---|---|---|---|---|---|---|")

    def cell(row, w):
        if w not in idx:
            return "-"
        return f"{row[idx[w]]} {units[idx[w]]}".strip()

    for row in r[2:]:
        name = row[idx["Kernel Name"]].split("(")[0].replace("(anonymous namespace)::", "")
        print(f"| `{name[:40]}` | {cell(row, 'gpu__time_duration.sum')} | {cell(row, 'dram__bytes_read.sum')} | "
              f"{cell(row, 'dram__bytes_write.sum')} | {cell(row, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
              f"{cell(row, 'sm__warps_active.avg.pct_of_peak_sustained_active')} | "
              f"{cell(row, 'launch__registers_per_thread')} | {cell(row, 'launch__grid_size')} |")
    print()


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def traffic(path, out_json, config):
    """DRAM bytes read + written per launch, first capture of each kernel (the
    roofline.traffic figure bench.py reports)."""
    import json

    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    ik, ir, iw = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    d = {}
    for row in r[2:]:
        name = row[ik].split("(")[0].replace("(anonymous namespace)::", "").split("::")[-1].split("<")[0].strip()
        name = name.replace("void ", "")
        if name in d:
            continue
        b = float(row[ir].replace(",", "")) * _SCALE[units[ir]] + float(row[iw].replace(",", "")) * _SCALE[units[iw]]
        d[name] = b
    json.dump({"config": config, "source": "ncu --set full --clock-control none, solve-only capture "
               "(profiles/prof_solve.py): " + os.path.basename(path), "dram_bytes_per_launch": d},
              open(out_json, "w"), indent=1)


if __name__ == "__main__":
    launches(sys.argv[1])
    if len(sys.argv) > 2:
        full(sys.argv[2])
    if len(sys.argv) > 4:
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
