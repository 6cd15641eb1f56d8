"""Summarise ncu output into profiles/: launch-list shares and full-set metrics per kernel.

    python scripts/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
    python scripts/ncu_summary.py full gpurun_out/prof.ncu-rep --config frames30 --E <E_slots> > profiles/rNN_ncu_full.md
        (also writes profiles/ncu_summary.json used by bench.py's roofline.traffic)
"""
import argparse
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    name = name.replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return name.split("(")[0].replace("void ", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ms": 1e3, "us": 1.0, "ns": 1e-3, "s": 1e6}.get(r[ui], 1.0)
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
    print(f"{sum(v[0] for v in agg.values())} launches, {tot/1e3:.2f} ms total\n")
    print("| kernel | launches | total ms | share | avg us |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {v[0]} | {v[1]/1e3:.3f} | {100*v[1]/tot:.1f}% | {v[1]/v[0]:.1f} |")


METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
]


def to_bytes(v, unit):
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1.0)


def full(rep, config, E, quiet=False):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary ({os.path.basename(rep)})\n")
    summary = {}
    for r in rows[2:]:
        name = short(r[hdr.index("Kernel Name")])
        rec = {}
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                rec[key] = (r[i], units[i])
        if not quiet:
            print(f"## {name}\n\n| metric | value |\n|---|---|")
            for key, label in METRICS:
                if key in rec:
                    print(f"| {label} | {rec[key][0]} {rec[key][1]} |")
        rd = to_bytes(float(rec["dram__bytes_read.sum"][0].replace(",", "")), rec["dram__bytes_read.sum"][1])
        wr = to_bytes(float(rec["dram__bytes_write.sum"][0].replace(",", "")), rec["dram__bytes_write.sum"][1])
        if not quiet:
            print(f"| DRAM read+write per launch | {(rd + wr)/1e9:.3f} GB |\n")
        kind = "ray_messages" if "ray_msg" in name else ("voxel_sum" if "reduce" in name else name)
        summary.setdefault(kind, {"config": config, "E": E, "dram_bytes_per_launch": 0.0, "launches": []})
        summary[kind]["launches"].append({"kernel": name, "dram_bytes": rd + wr})
    # one K5 "launch" in bench.py = all length classes of one iteration: sum the LAST launch of
    # each class kernel (the capture spans whole iterations)
    for kind, s in summary.items():
        per = {}
        for l in s["launches"]:
            per[l["kernel"]] = l["dram_bytes"]
        s["dram_bytes_per_launch"] = sum(per.values())
        s["launches"] = [{"kernel": k, "dram_bytes": v} for k, v in per.items()]
    json.dump({"kernels": summary}, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("path")
    ap.add_argument("--config", default="frames30")
    ap.add_argument("--E", type=int, default=0)
    ap.add_argument("--quiet", action="store_true", help="only write profiles/ncu_summary.json")
    a = ap.parse_args()
    launches(a.path) if a.mode == "launches" else full(a.path, a.config, a.E, a.quiet)
