#!/usr/bin/env python
"""Per-source-line instruction and stall-sample shares of one kernel in an
.ncu-rep (needs -lineinfo and --import-source on):
    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def page(rep, src):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", src],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    addr2line, line = {}, None
    fname = None
    for r in page(rep, "cuda,sass"):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) >= 4 and r[0].isdigit():
            line = (fname, int(r[0]), r[1].strip()[:70])
        if len(r) >= 4 and r[2].startswith("0x"):
            addr2line[r[2]] = line
    rows = page(rep, "sass")
    hdr = rows[1]
    ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    inst, stall = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= max(ie, st):
            continue
        l = addr2line.get(r[0])
        inst[l] += int(r[ie] or 0)
        stall[l] += int(r[st] or 0)
    ti, ts = sum(inst.values()), sum(stall.values())
    print(f"warp instructions {ti}, stall samples {ts}")
    for l, n in inst.most_common(top):
        print(f"{100 * n / ti:5.1f}% inst {100 * stall[l] / ts:5.1f}% stall  {l}")


if __name__ == "__main__":
    main()
