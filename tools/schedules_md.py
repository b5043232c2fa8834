#!/usr/bin/env python
"""Render the tables of profiles/<round>/schedules.md from tools/schedules.py's
JSON (the prose between them is kept from the existing file):
    python tools/schedules_md.py gpurun_out/schedules.json profiles/r01/schedules.md"""
import json
import re
import sys


def host_table(d):
    rows = ["| schedule | transfers/frame | H2D ms | kernel ms | D2H ms | transfer share | y share of kernels "
            "| total ms | frames/s |", "|---|---|---|---|---|---|---|---|---|"]
    for name, label in (("naive", "naive"), ("optimized", "optimized"), ("fused", "fused"),
                        ("streamed", "streamed (overlapped, chunked)")):
        s = d[name]
        tpf = (s["h2d_count"] + s["d2h_count"]) / s["frames"]
        if name == "streamed":
            rows.append(f"| {label} | {tpf:.2f} | - | - | - | - | - | {s['total_ms']:.2f} | {s['fps']:.0f} |")
            continue
        ys = f"{100 * s['y_share_of_kernels']:.1f}%" if "y_share_of_kernels" in s else "-"
        rows.append(f"| {label} | {tpf:.0f} | {s['h2d_ms']:.2f} | {s['kernel_ms']:.2f} | {s['d2h_ms']:.2f} | "
                    f"{100 * s['share_transfers']:.1f}% | {ys} | {s['total_ms']:.2f} | {s['fps']:.0f} |")
    t = d["tuning_effect"]
    rows.append("")
    rows.append(f"Tuning (naive -> optimised): H2D bytes -{100 * t['h2d_byte_reduction']:.1f}%, time "
                f"-{100 * t['h2d_time_reduction']:.1f}%; D2H bytes -{100 * t['d2h_byte_reduction']:.1f}%, time "
                f"-{100 * t['d2h_time_reduction']:.1f}%; kernel time x{t['kernel_time_ratio_opt_over_naive']:.2f}; "
                f"total speed-up {t['speedup_opt_over_naive']:.2f}x. Fused per-frame loop: "
                f"{t['speedup_fused_over_opt']:.2f}x over optimised; overlapped stream: "
                f"{t['speedup_streamed_over_opt']:.1f}x over optimised.")
    return "\n".join(rows)


def device_table(j):
    rows = ["| stream | fused ms | unfused ms (H + V) | speed-up | required bytes unfused/fused | fused GB/s "
            "| unfused GB/s | bit-exact |", "|---|---|---|---|---|---|---|---|"]
    for k in sorted(x for x in j if x.startswith("device_ab_")):
        d = j[k]
        rows.append(f"| {d['frames']} x {d['w']}x{d['h']} {d['chroma']} | {d['fused_ms']:.3f} | "
                    f"{d['unfused_ms']:.3f} ({d['htask_ms']:.3f} + {d['vtask_ms']:.3f}) | "
                    f"{d['speedup_fused']:.2f}x | {d['byte_ratio']:.3f} | {d['fused_gbs']:.0f} | "
                    f"{d['unfused_gbs']:.0f} | {d['bit_exact']} |")
    return "\n".join(rows)


def replace_table(md, heading, table):
    """Replace the first markdown table (and an immediately following 'Tuning' line) after heading."""
    i = md.index(heading)
    j = md.index("\n|", i) + 1
    k = j
    lines = md[j:].split("\n")
    n = 0
    while n < len(lines) and lines[n].startswith("|"):
        n += 1
    end = j + sum(len(x) + 1 for x in lines[:n])
    if md[end:].startswith("\nTuning"):
        end = md.index("\n", end + 1) + 1
    return md[:k] + table + "\n" + md[end:]


def main():
    j = json.load(open(sys.argv[1]))
    path = sys.argv[2]
    md = open(path).read()
    md = replace_table(md, "## CIF 352x288 4:2:0, 2000 frames", host_table(j["host_schedules_cif_2000"]))
    md = replace_table(md, "## HD 1920x1080 4:2:0, 300 frames", host_table(j["host_schedules_hd_300"]))
    md = replace_table(md, "## Device-resident A/B", device_table(j))
    open(path, "w").write(md)


if __name__ == "__main__":
    main()
