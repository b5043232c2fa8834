#!/usr/bin/env python
"""Summarise ncu output brought back in gpurun_out/ into profiles/.

    python tools/ncu_summary.py --round r01 [--launches gpurun_out/launches.csv]
                                [--rep hd420=gpurun_out/prof_hd420.ncu-rep ...]

Writes profiles/<round>/ncu_launches.md (per-kernel share of the launch list),
profiles/<round>/ncu_full_<cfg>.txt (selected --set full metrics) and merges
per-launch DRAM traffic into profiles/ncu_summary.json, which bench.py reads
for roofline.traffic.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_bytes.sum",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    per = defaultdict(lambda: [0, 0.0])
    order = []
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(unit, 1)
        name = r["Kernel Name"]
        short = name.split("(")[0]
        per[short][0] += 1
        per[short][1] += us
        order.append((short, us))
    return per, order


def raw_metrics(rep):
    out = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        res.append(d)
    return res


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def scale(v, u):
    f = to_float(v)
    if f is None:
        return None
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
                "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r01")
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--note", default="")
    ap.add_argument("--build", default="", help="library source hash the captures were made on "
                                                  "(default: the current tree's, bench.source_hash)")
    ap.add_argument("--frames", type=int, action="append", default=[],
                    help="frames per profiled launch, one per --rep (default: bench defaults)")
    a = ap.parse_args()
    outdir = os.path.join(ROOT, "profiles", a.round)
    os.makedirs(outdir, exist_ok=True)

    if os.path.exists(a.launches):
        per, order = launches(a.launches)
        tot = sum(v[1] for v in per.values())
        lines = [f"# ncu launch list ({a.round})", "",
                 "`ncu --metrics gpu__time_duration.sum --clock-control none` over the default",
                 "`python bench.py` command (cold-cache, serialised launches: compare SHARES).", "",
                 "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
        for k, (n, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {n} | {us:.1f} | {us / n:.2f} | {100 * us / tot:.1f}% |")
        lines += ["", f"total launches: {sum(v[0] for v in per.values())}; total {tot:.1f} us"]
        if a.note:
            lines += ["", a.note]
        open(os.path.join(outdir, "ncu_launches.md"), "w").write("\n".join(lines) + "\n")
        print("\n".join(lines))

    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    for ri, spec in enumerate(a.rep):
        cfg, rep = spec.split("=", 1)
        frames = a.frames[ri] if ri < len(a.frames) else (1000 if cfg.startswith("4k") else 300)
        ms = raw_metrics(rep)
        txt = [f"# ncu --set full: {os.path.basename(rep)} ({a.round}, config {cfg})"]
        for i, d in enumerate(ms):
            name = d.get("Kernel Name", ("?", ""))[0]
            txt.append(f"\n## launch {i}: {name}")
            for k in KEEP:
                if k in d:
                    txt.append(f"{k} [{d[k][1]}] = {d[k][0]}")
            stalls = sorted(((to_float(v[0]) or 0.0, k) for k, v in d.items()
                             if k.startswith("smsp__average_warps_issue_stalled_") and
                             k.endswith("_per_issue_active.ratio")), reverse=True)[:8]
            txt.append("top stall reasons (warps per issue):")
            for v, k in stalls:
                txt.append(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.3f}")
        open(os.path.join(outdir, f"ncu_full_{cfg}.txt"), "w").write("\n".join(txt) + "\n")
        print("\n".join(txt))
        d = ms[0]
        rd = scale(*d["dram__bytes_read.sum"])
        wr = scale(*d["dram__bytes_write.sum"])
        dur = scale(*d["gpu__time_duration.sum"])
        import sys

        sys.path.insert(0, ROOT)
        import bench

        summ[cfg] = {"dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
                     "duration_us_under_ncu": dur, "frames_per_launch": frames,
                     "build_sha": a.build or bench.source_hash(),
                     "source": f"profiles/{a.round}/ncu_full_{cfg}.txt (ncu --set full --clock-control none)"}
    if a.rep:
        json.dump(summ, open(summ_path, "w"), indent=1)


if __name__ == "__main__":
    main()
