#!/usr/bin/env python
"""SURVEY f3 measurement: K-N1g (fused band kernel, any spec) on the HD
stream, against K-N2 (per-pixel literal kernel) on the same spec, and against
K-N1 on SPEC's own taps.

    python tools/general_perf.py [--out gpurun_out/general_perf.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1103_4881_b200 as ds

# a longer Array-OL downscaler reading: 13-tap H / 14-tap V windows
HALO_H = dict(pattern=13, paving=8, origin=-2,
              weights=[[1, 3, 5, 3, 1, 0, 0, 0, 0, 0, 0, 0, 0], [0, 0, 0, 1, 3, 5, 3, 1],
                       [0, 0, 0, 0, 0, 0, 1, 3, 5, 3, 1]], divisor=13, bias=6)
HALO_V = dict(pattern=14, paving=9, origin=-2,
              weights=[[1, 2, 4, 2, 1], [0, 0, 1, 2, 4, 2, 1], [0, 0, 0, 0, 0, 1, 2, 4, 2, 1],
                       [0, 0, 0, 0, 0, 0, 0, 0, 1, 2, 4, 2, 1]], divisor=10, bias=5)


def timed(fn, steps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def run(W, H, n, spec, kernels, steps=20, run_bands=0):
    d = ds.Downscaler(W, H, 3, spec=spec)
    d.set_run_bands(run_bands)
    x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
    outs, res = {}, {}
    for k in kernels:
        d.set_kernel(k)
        y = d.alloc_out(n)
        ms = timed(lambda: d(x, y), steps if k != ds.DS_KERNEL_GENERIC else 3)
        assert d.last_kernel() == k
        outs[k] = y
        fb = n * (d.in_frame_bytes + d.out_frame_bytes)
        res[ds.KERNEL_NAMES[k]] = {"ms": ms, "fps": n / ms * 1e3, "in_plus_out_gbs": fb / ms / 1e6}
    ref = outs[kernels[0]]
    res["all_kernels_bit_identical"] = all(torch.equal(ref, o) for o in outs.values())
    p = d.plan
    res["k1g_bands"] = list(p.general_band_reps)
    res["k1g_staged_bytes_max"] = p.general_stage_bytes_max
    return res


def generic_task(n=300, W=1920, H=1080):
    """The paper's yhfk H task over n HD luma planes as ONE 3-D Array-OL task
    (frames are a repetition dimension), through ds_run_task (both launch
    policies) vs the dedicated unfused H-task kernel (K-N3)."""
    x = ds.generate_frames(n, W * H, seed=1)
    mid = torch.empty((n, H, W // 8 * 3), dtype=torch.uint8, device="cuda")
    mid2 = torch.empty_like(mid)
    spec = ds.ds_default_spec()
    hw = [[spec.h.weight[k][i] for i in range(8)] for k in range(3)]
    tin = ds.make_tiler((n, H, W), (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, 8]], [[0], [0], [1]], [8])
    tout = ds.make_tiler((n, H, W // 8 * 3), (0, 0, 0), [[1, 0, 0], [0, 1, 0], [0, 0, 3]],
                         [[0], [0], [1]], [3])
    body = ds.make_body(hw, 6, 3, n_in=8)
    res = {}
    for pol, name in ((ds.DS_TOPO_FLAT, "flat"), (ds.DS_TOPO_SPEC, "spec_topology")):
        ms = timed(lambda: ds.run_task(x, tin, mid, tout, [n, H, W // 8], body, policy=pol), 5)
        res[f"ds_run_task_{name}_ms"] = ms
    # the same task with the input origin shifted by 3 columns: windows wrap at
    # the row end, so the tiler is not affine -> the modulo path
    tin_w = ds.make_tiler((n, H, W), (0, 0, 3), [[1, 0, 0], [0, 1, 0], [0, 0, 8]], [[0], [0], [1]], [8])
    mid_w = torch.empty_like(mid)                # its own buffer: different results
    res["ds_run_task_wrapping_origin_ms"] = timed(
        lambda: ds.run_task(x, tin_w, mid_w, tout, [n, H, W // 8], body), 5)
    d = ds.Downscaler(W, H, 1)
    res["htask_kernel_ms"] = timed(lambda: d.htask(x, mid2), 20)
    res["bit_identical"] = bool(torch.equal(mid, mid2))
    res["bytes"] = n * W * H * (1 + 3 / 8)
    res["ds_run_task_flat_gbs"] = res["bytes"] / res["ds_run_task_flat_ms"] / 1e6
    res["htask_kernel_gbs"] = res["bytes"] / res["htask_kernel_ms"] / 1e6
    return res


def generic_vtask(n=300, W=1920, H=1080):
    """The paper's V task over n HD luma Mid planes (H rows x 3W/8) as ONE 3-D
    Array-OL task (repetition (n, H/9, 3W/8); input pattern 9 rows down a
    column, output pattern 4 rows), through ds_run_task vs K-N3's V kernel."""
    Wm, Ho = W // 8 * 3, H // 9 * 4
    mid = ds.generate_frames(n, H * Wm, seed=2).view(n, H, Wm)
    out = torch.empty((n, Ho, Wm), dtype=torch.uint8, device="cuda")
    spec = ds.ds_default_spec()
    vw = [[spec.v.weight[k][i] for i in range(9)] for k in range(4)]
    tin = ds.make_tiler((n, H, Wm), (0, 0, 0), [[1, 0, 0], [0, 9, 0], [0, 0, 1]], [[0], [1], [0]], [9])
    tout = ds.make_tiler((n, Ho, Wm), (0, 0, 0), [[1, 0, 0], [0, 4, 0], [0, 0, 1]], [[0], [1], [0]], [4])
    body = ds.make_body(vw, 8, 4, n_in=9)
    res = {}
    for pol, name in ((ds.DS_TOPO_FLAT, "flat"), (ds.DS_TOPO_SPEC, "spec_topology")):
        res[f"ds_run_task_{name}_ms"] = timed(lambda: ds.run_task(mid, tin, out, tout, [n, H // 9, Wm], body,
                                                                  policy=pol), 5)
    ref = out.clone()
    d = ds.Downscaler(W, H, 1)
    out2 = torch.empty_like(out)
    res["vtask_kernel_ms"] = timed(lambda: d.vtask(mid.view(n, -1), out2.view(n, -1)), 20)
    res["bit_identical"] = bool(torch.equal(ref, out2))
    res["bytes"] = n * (H * Wm * 8 // 9 + Ho * Wm)
    res["ds_run_task_flat_gbs"] = res["bytes"] / res["ds_run_task_flat_ms"] / 1e6
    res["vtask_kernel_gbs"] = res["bytes"] / res["vtask_kernel_ms"] / 1e6
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/general_perf.json")
    ap.add_argument("--quick", action="store_true", help="K-N1g only, one line per spec")
    ap.add_argument("--run-bands", type=int, default=0, help="K-N1g bands per run (0 = automatic)")
    ap.add_argument("--tasks", action="store_true", help="general task executor only (H and V tasks)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    halo = ds.make_spec(h=HALO_H, v=HALO_V)
    if a.tasks:
        print(json.dumps({"h": generic_task(), "v": generic_vtask()}))
        return
    if a.quick:
        h = run(1920, 1080, 300, halo, [ds.DS_KERNEL_FUSED_GENERAL], steps=50, run_bands=a.run_bands)
        t = run(1920, 1080, 300, None, [ds.DS_KERNEL_FUSED_GENERAL], steps=50)
        k = ds.KERNEL_NAMES[ds.DS_KERNEL_FUSED_GENERAL]
        print(json.dumps({"halo_ms": round(h[k]["ms"], 4), "spec_taps_ms": round(t[k]["ms"], 4)}))
        return
    out = {
        "gpu": torch.cuda.get_device_name(0),
        "halo_spec": {"h": HALO_H, "v": HALO_V},
        "hd420_300_halo_spec": run(1920, 1080, 300, halo,
                                   [ds.DS_KERNEL_FUSED_GENERAL, ds.DS_KERNEL_GENERIC]),
        "hd420_300_spec_taps": run(1920, 1080, 300, None,
                                   [ds.DS_KERNEL_FUSED, ds.DS_KERNEL_FUSED_GENERAL]),
        "generic_task_yhfk_300_hd_luma": generic_task(),
        "generic_task_v_300_hd_luma": generic_vtask(),
    }
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
