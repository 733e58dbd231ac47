#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv]
                                --out profiles/r01 [--events 100000000] [--config 100M]

Writes <out>_kernels.md (per-kernel DRAM bytes, time, achieved GB/s, occupancy,
instructions, top stall reasons from the --set full capture), <out>_launches.md
(per-kernel share of one step from the gpu__time_duration launch list) and
updates profiles/traffic.json with the per-launch DRAM traffic of k_onesweep
(bench.py reports it as roofline.traffic).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, [dict(zip(hdr, r)) for r in rows[2:]]


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def base_name(k):
    k = k.replace("void ", "").replace("pm4g::", "")
    name = k.split("(")[0]
    if name.startswith("k_onesweep_pf<") or name.startswith("k_onesweep_pf0<"):   # persistent log-sort passes
        return "k_onesweep"
    if name.startswith("k_onesweep<"):   # log-sort passes carry the u8/u16 activity; u32 = small sorts
        return "k_onesweep" if "unsigned int" not in name.split(",")[0] else "k_onesweep_small"
    return name.split("<")[0]


def kernels_md(rep, events):
    hdr, units, rows = raw_rows(rep)
    u = dict(zip(hdr, units))
    stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")]
    lines = ["| kernel | ms | DRAM read GB | DRAM write GB | DRAM GB/s | B/event | warps active % | regs | occ limit (regs/smem) | warp-instr | top stalls (per issue) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    per = defaultdict(list)
    for r in rows:
        ms = num(r["gpu__time_duration.sum"]) * {"usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6}.get(
            u.get("gpu__time_duration.sum"), 1.0)
        scale = lambda h: {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u.get(h, ""), 1.0)  # noqa: E731
        rd = num(r["dram__bytes_read.sum"]) * scale("dram__bytes_read.sum")
        wr = num(r["dram__bytes_write.sum"]) * scale("dram__bytes_write.sum")
        st = sorted(((num(r[h]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for h in stall), reverse=True)[:3]
        name = base_name(r["Kernel Name"])
        per[name].append((rd + wr) * 1e9)
        lines.append(f"| {name} | {ms:.3f} | {rd:.3f} | {wr:.3f} | {(rd + wr) / (ms / 1e3):.0f} | "
                     f"{(rd + wr) * 1e9 / events:.1f} | {num(r['sm__warps_active.avg.pct_of_peak_sustained_active']):.0f} | "
                     f"{r.get('launch__registers_per_thread', '')} | {r.get('launch__occupancy_limit_registers', '')}/"
                     f"{r.get('launch__occupancy_limit_shared_mem', '')} | {num(r['smsp__inst_executed.sum']) / 1e6:.0f} M | "
                     + ", ".join(f"{n} {v:.2f}" for v, n in st) + " |")
    return "\n".join(lines), per


def launches_md(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        v = num(d["Metric Value"])
        unit = d["Metric Unit"]
        ms = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1e-6)
        k = base_name(d["Kernel Name"])
        if not k.startswith("k_"):   # the workload generator's torch kernels are not part of the step
            continue
        agg[k][0] += 1
        agg[k][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")
    lines.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% |")
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--events", type=float, default=1e8)
    ap.add_argument("--config", default="100M")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    traffic = {}
    if a.rep:
        md = [f"# ncu --set full summary ({a.config}, {a.events:.0f} events per launch input)", "", a.note, ""]
        for rep in a.rep:
            t, per = kernels_md(rep, a.events)
            md += [f"## {os.path.basename(rep)}", "", t, ""]
            for k, v in per.items():
                traffic.setdefault(k, []).extend(v)
        open(a.out + "_kernels.md", "w").write("\n".join(md) + "\n")
    if a.launches:
        md = [f"# Launch list (ncu gpu__time_duration.sum, --clock-control none): {a.config}", "",
              "Cold-cache and serialised per launch: compare shares, not absolutes.  libpm4g kernels",
              "only (k_*); the synthetic generator's torch kernels in the same process are excluded.", "",
              a.note, "",
              launches_md(a.launches)]
        open(a.out + "_launches.md", "w").write("\n".join(md) + "\n")
    if traffic:
        tf = os.path.join(os.path.dirname(a.out) or ".", "traffic.json")
        cur = json.load(open(tf)) if os.path.exists(tf) else {}
        for k, v in traffic.items():
            cur[k] = {"config": a.config, "dram_bytes_per_launch": sum(v) / len(v), "launches_captured": len(v),
                      "source": os.path.basename(a.out)}
        json.dump(cur, open(tf, "w"), indent=1)


if __name__ == "__main__":
    main()
