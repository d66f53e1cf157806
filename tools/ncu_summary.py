#!/usr/bin/env python
"""Summarise ncu captures for profiles/: key metrics per kernel (from an
--set full .ncu-rep) and launch shares (from a --metrics gpu__time_duration
csv launch list).  Usage:
  python tools/ncu_summary.py REP.ncu-rep LAUNCHES.csv OUT.md [frames_per_launch] [captured command]
Also writes profiles/r2_traffic.json (DRAM bytes of the census kernels of one
launch, summed) for bench.py's roofline.traffic."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe % (POPC)"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU data-pipe wavefronts % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def stalls(rep, kernel_regex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel_regex}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h = rows[1]
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    tot = collections.Counter()
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        for c in cols:
            try:
                tot[c[6:]] += float(r[h.index(c)] or 0)
            except ValueError:
                pass
    s = sum(tot.values()) or 1
    return {k: round(100 * v / s, 1) for k, v in tot.most_common(6)}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"].split("(")[0].split("::")[-1]].append(float(d["Metric Value"]))
    return agg


def main():
    rep, lcsv, out = sys.argv[1:4]
    fpl = int(sys.argv[4]) if len(sys.argv) > 4 else 32
    cmd = sys.argv[5] if len(sys.argv) > 5 else f"bench.py --frames {fpl}"
    data, units = raw(rep)
    lines = [f"# ncu summary: {os.path.basename(rep)}", "",
             f"Capture: `ncu --set full --clock-control none --import-source on` of "
             f"`{cmd}` (one launch per kernel shown; one launch = {fpl} C2 frames).", ""]
    traffic = {"census_dram_bytes_per_launch": 0.0, "frames_per_launch": fpl, "per_kernel": {}}
    for d in data:
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for m, label in METRICS:
            if m in d:
                lines.append(f"| {label} (`{m}`) | {d[m]} {units.get(m, '')} |")
        st = stalls(rep, name)
        if st:
            lines.append(f"| top stall reasons (% of samples) | {', '.join(f'{k} {v}' for k, v in st.items())} |")
        lines.append("")
        if "census" in name:
            sc = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = sum(float(d[m].replace(",", "")) * sc.get(units.get(m, "byte"), 1.0)
                    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            key = name + " " + d.get("Grid Size", d.get("launch__grid_size", ""))
            if key not in traffic["per_kernel"]:  # one launch of each kernel (the capture may hold two batches)
                traffic["census_dram_bytes_per_launch"] += b
                traffic["per_kernel"][key] = b
            traffic["source"] = f"{os.path.basename(rep)}: {cmd}"
    if lcsv and os.path.exists(lcsv):
        agg = launches(lcsv)
        tot = sum(sum(v) for v in agg.values())
        lines += ["## launch list (all launches of the run, cold-cache serialised)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {k} | {len(v)} | {sum(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    if traffic["census_dram_bytes_per_launch"]:
        json.dump(traffic, open(os.path.join(os.path.dirname(out), "r2_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
