#!/usr/bin/env python
"""Benchmark of the B200 downscaler (arxiv 1103.4881 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config hd420|hd444|4k420|4k444|cif420|sd420|qcif420]
                    [--spec spec|halo] [--frames F] [--no-verify] [--ncu|--no-ncu]

One step = one ds_run over the whole per-rank batch of frames (every row of
SURVEY 8(a): H task -> u8 intermediate -> V task, all planes, all frames)
with the input already resident in HBM.  N = 1 runs BASELINE configs[2]
(300-frame HD 4:2:0 stream on one B200); N > 1 (torchrun) weak-scales it,
300 frames per GPU frame-sharded by global index (--frames 3000 runs
configs[3]'s fixed 3000-frame stream instead).  --spec halo runs the same
stream through a 13/14-tap filter with halos and origins -2 (the K-N1g
kernel).  Rank 0 prints ONE JSON line.
"Measurement" for every field.

Legs besides the timed region: e2e (ds_run_host from pinned host memory),
every-frame parity of the output stream against the CPU oracle on all host
cores (oracle/verify.py; rank 0 checks the gathered stream at N > 1), the
cpu_baseline (the oracle on one pinned core), an in-run ncu capture of one
launch for roofline.traffic (N = 1), and at N > 1 the gather to rank 0
(NCCL), the gather fused into the kernels' stores (peer memory), and a
1-GPU solo run of the same per-GPU workload for speedup_vs_1gpu.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import shutil
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("frames/s and achieved HBM GB/s (% of B200 peak) at 1/2/4/8 GPUs vs CPU oracle")

CONFIGS = {
    "hd420": dict(w=1920, h=1080, channels=3, chroma=1, label="HD 1920x1080 YUV 4:2:0"),
    "hd444": dict(w=1920, h=1080, channels=3, chroma=0, label="HD 1920x1080 YUV 4:4:4"),
    "4k420": dict(w=3840, h=2160, channels=3, chroma=1, label="4K 3840x2160 YUV 4:2:0"),
    "4k444": dict(w=3840, h=2160, channels=3, chroma=0, label="4K 3840x2160 YUV 4:4:4"),
    "cif420": dict(w=352, h=288, channels=3, chroma=1, label="CIF 352x288 YUV 4:2:0"),
    # rows that are not 16-byte multiples (chroma 360 / 88 B)
    "sd420": dict(w=720, h=576, channels=3, chroma=1, label="PAL SD 720x576 YUV 4:2:0"),
    "qcif420": dict(w=176, h=144, channels=3, chroma=1, label="QCIF 176x144 YUV 4:2:0"),
}

# Filter specs.  "spec": SPEC's downscaler (hfilter_8to3 S:530, vfilter_9to4
# S:540), the default.  "halo": a longer 8->3 / 9->4 downscaler whose input
# patterns overlap (P = 13 > S = 8 horizontally, 14 > 9 vertically) with
# origins -2, so every band stages its filter halo and windows wrap
# toroidally at the plane edges: the K-N1g path.
HALO_SPEC = (
    dict(pattern=13, paving=8, origin=-2, weights=[[1, 3, 5, 3, 1], [0, 0, 0, 1, 3, 5, 3, 1],
                                                    [0, 0, 0, 0, 0, 0, 1, 3, 5, 3, 1]],
         divisor=13, bias=6),
    dict(pattern=14, paving=9, origin=-2, weights=[[1, 2, 4, 2, 1], [0, 0, 1, 2, 4, 2, 1],
                                                    [0, 0, 0, 0, 0, 1, 2, 4, 2, 1],
                                                    [0, 0, 0, 0, 0, 0, 0, 0, 1, 2, 4, 2, 1]],
         divisor=10, bias=5),
)
SPECS = {"spec": None, "halo": HALO_SPEC}
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback, only if MEASURED_PEAKS.json is absent
CLOCK_WINDOW_MS = 25.0      # clock-sampled replays on each side of the timed region


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="hd420")
    ap.add_argument("--spec", choices=sorted(SPECS), default="spec",
                    help="filter spec: SPEC's downscaler (default) or the halo spec (K-N1g)")
    ap.add_argument("--frames", type=int, default=0,
                    help="TOTAL frames (strong scaling); default: 300 HD / 1000 4K frames "
                         "per GPU (weak scaling)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--kernel", choices=["auto", "fused", "fused_general", "generic"], default="auto")
    ap.add_argument("--band-bytes", type=int, default=0, help="K-N1 band size (0 = default)")
    ap.add_argument("--graph", dest="graph", action="store_true", default=True,
                    help="(default) capture the K timed ds_run calls in one CUDA graph and time one "
                         "replay: every step is still a full launch over the batch, without host "
                         "launch gaps or per-step event records between them")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time each ds_run between its own CUDA events (per-launch median / best)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU-oracle sample budget (seconds of 1-core work)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-verify", action="store_true",
                    help="skip the every-frame oracle check of the output stream")
    ap.add_argument("--ncu", dest="ncu", action="store_true", default=None,
                    help="measure roofline.traffic in-run: ncu on one launch in a child process "
                         "(default at N = 1 when ncu is on PATH)")
    ap.add_argument("--no-ncu", dest="ncu", action="store_false")
    ap.add_argument("--gather-reps", type=int, default=5, help="N>1: timed gathers (after one warm-up)")
    ap.add_argument("--no-gather", action="store_true", help="N>1: skip the gather legs")
    ap.add_argument("--fused-gather", dest="fused_gather", action="store_true", default=None,
                    help="N>1: time ds_run storing straight into rank 0's buffer (default: on when "
                         "a one-process peer-store probe passes)")
    ap.add_argument("--no-fused-gather", dest="fused_gather", action="store_false")
    ap.add_argument("--no-solo", action="store_true", help="N>1: skip the 1-GPU solo run")
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--peer-probe", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args(argv)


def workload(args, world):
    """Frames per run.  Default: weak scaling, 300 HD frames per GPU (N = 1 is
    configs[2] exactly; frames are independent, so ranks share no data
    path).  --frames F fixes the TOTAL instead (strong scaling; --frames 3000
    is configs[3] literally)."""
    cfg = dict(CONFIGS[args.config])
    per_gpu = 1000 if args.config.startswith("4k") else 300
    if args.frames:
        total, scaling = args.frames, ("weak" if world == 1 else "strong")
    else:
        total, scaling = per_gpu * world, "weak"
    cfg["total"] = total
    cfg["scaling"] = scaling
    if args.config.startswith("hd") and world == 1 and total == 1:
        cfg["name"] = f"configs[1]: one {cfg['label']} frame on 1 B200 (latency; L2-resident)"
    elif args.config.startswith("hd") and world == 1 and total == 300:
        cfg["name"] = f"configs[2]: 300-frame {cfg['label']} stream on 1 B200"
    elif args.config.startswith("hd") and not args.frames:
        cfg["name"] = (f"configs[2] per GPU, weak-scaled: {total}-frame {cfg['label']} stream "
                       f"frame-sharded over {world} B200 (300 frames per GPU; configs[3] scale)")
    elif args.config.startswith("hd") and total == 3000:
        cfg["name"] = f"configs[3]: 3000-frame {cfg['label']} stream frame-sharded over {world} B200"
    elif args.config.startswith("4k") and total == 1000 * max(1, world) and not args.frames:
        cfg["name"] = (f"configs[4] per GPU, weak-scaled: {total}-frame {cfg['label']} stream over "
                       f"{world} B200")
    elif args.config.startswith("4k") and total == 1000:
        cfg["name"] = f"configs[4]: 1000-frame {cfg['label']} stream over {world} B200"
    else:
        cfg["name"] = f"{total}-frame {cfg['label']} stream over {world} B200"
    if getattr(args, "spec", "spec") != "spec":
        cfg["name"] += f", {args.spec} filter spec"
    return cfg


def spec_stages(args):
    """(h, v) stage dicts of --spec, or None for SPEC's downscaler."""
    return SPECS[getattr(args, "spec", "spec")]


def geometry(cfg, stages=None):
    """(in, out, required-in) bytes per frame.  Out planes are
    (Q_h W/S_h) x (Q_v H/S_v) (3W/8 x 4H/9 for both specs here).
    Required input: with SPEC's taps input rows 9g+4 carry zero V weight
     and are never needed, 8/9 of the input; the halo spec reads every
    row (each row lies in some pattern's live taps)."""
    import synth

    dims = synth.plane_dims(cfg["w"], cfg["h"], cfg["channels"], cfg["chroma"])
    if stages is None:
        qh, sh, qv, sv = 3, 8, 4, 9
    else:
        h, v = stages
        qh, sh, qv, sv = len(h["weights"]), h["paving"], len(v["weights"]), v["paving"]
    fin = sum(w * h for w, h in dims)
    fout = sum((qh * w // sh) * (qv * h // sv) for w, h in dims)
    fin_req = fin * 8 // 9 if stages is None else fin
    return fin, fout, fin_req


def config_dict(args, cfg, world, n_rank=None):
    """The `config` object, identical in both arms (same keys and values)."""
    fin, fout, _ = geometry(cfg, spec_stages(args))
    per = -(-cfg["total"] // world) if world else cfg["total"]
    return {
        "workload": cfg["name"], "frames": cfg["total"], "frames_per_rank_max": per,
        "w": cfg["w"], "h": cfg["h"], "channels": cfg["channels"],
        "chroma": "4:2:0" if cfg["chroma"] else "4:4:4",
        "spec": args.spec if args.spec != "spec" else "SPEC downscaler (S:530, S:540)",
        "in_frame_bytes": fin, "out_frame_bytes": fout,
        "parallelism": f"frame-sharded x{world}" if world > 1 else "single GPU",
        "l2": f"inputs larger than L2: {per * (fin + fout) / 1e9:.3f} GB touched per step per GPU "
              f"vs 126 MB L2 (no flush needed)",
    }


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def source_hash():
    """sha256 (16 hex) of the library sources: stamps ncu captures so a kernel
    change shows up as a stale roofline.traffic."""
    import glob

    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_1103_4881_b200", "csrc", "*")) +
                   [os.path.join(ROOT, "include", "ds.h")])
    for f in files:
        if f.endswith((".cu", ".cuh", ".h")):
            with open(f, "rb") as fh:
                h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons every ~1 ms DURING the
    timed region (and the clock windows around it)."""

    REASONS = {
        0x0000000000000001: "gpu_idle", 0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap", 0x0000000000000008: "hw_slowdown",
        0x0000000000000010: "sync_boost", 0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown", 0x0000000000000080: "hw_power_brake_slowdown",
        0x0000000000000100: "display_clock_setting",
    }

    def __init__(self, device_index: int, period_s: float = 0.001):
        self.samples, self.reasons, self.marks = [], set(), {}
        self.period = period_s
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.hdl = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.hdl, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.hdl, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.hdl)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def mark(self, name):
        self.marks[name] = len(self.samples)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def result(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        a, b = self.marks.get("timed_start", 0), self.marks.get("timed_end", len(self.samples))
        timed = self.samples[a:b]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons - {"gpu_idle"}),
                "samples": len(self.samples), "samples_in_timed_region": len(timed),
                "sm_mhz_timed_region": statistics.median(timed) if timed else None,
                "period_ms": self.period * 1e3,
                "window": f"sampled continuously over >= {CLOCK_WINDOW_MS:.0f} ms of the same step "
                          f"replayed on each side of the timed region and the region itself"}


def ncu_committed(config_key, frames_per_launch):
    """Per-launch DRAM bytes of the committed ncu --set full summary of this
    config (profiles/ncu_summary.json), scaled per frame; with the build
    stamp it was captured on, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            e = json.load(f)[config_key]
    except Exception:
        return None
    n0 = e.get("frames_per_launch", frames_per_launch)
    return {"traffic": e["dram_bytes_per_launch"] * frames_per_launch / n0,
            "dram_gbs": e["dram_bytes_per_launch"] / (e["duration_us_under_ncu"] * 1e-6) / 1e9,
            "source": e.get("source", "") + (f" (scaled from {n0} to {frames_per_launch} frames)"
                                             if n0 != frames_per_launch else ""),
            "build": e.get("build_sha")}


def ncu_measure(args, timeout_s=240):
    """roofline.traffic measured in this run: ncu (one child process, cold
    cache, clocks uncontrolled) on ONE launch of the same workload -- DRAM
    read + write bytes and its duration.  None if ncu is unavailable."""
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu")
                                  else None)
    if not ncu:
        return None, "ncu not found"
    child = [sys.executable, os.path.abspath(__file__), "--ncu-child", "--config", args.config,
             "--spec", args.spec, "--seed", str(args.seed), "--kernel", args.kernel]
    if args.frames:
        child += ["--frames", str(args.frames)]
    if args.band_bytes:
        child += ["--band-bytes", str(args.band_bytes)]
    if args.stages or args.ctas:
        child += ["--stages", str(args.stages), "--ctas", str(args.ctas)]
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--kernel-name", "regex:^ds_(fused|generic|spec)", "--launch-skip", "3",
           "--launch-count", "1", "--csv", *child]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout_s, cwd=ROOT)
    except Exception as e:
        return None, f"ncu failed: {e}"
    vals, kname = {}, None
    import csv
    import io

    text = r.stdout
    start = text.find('"ID"')
    if start < 0:
        return None, f"ncu rc={r.returncode}: {(r.stderr or r.stdout)[-300:]}"
    for row in csv.DictReader(io.StringIO(text[start:])):
        name, unit = row.get("Metric Name"), row.get("Metric Unit", "")
        try:
            v = float(row["Metric Value"].replace(",", ""))
        except Exception:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                 "second": 1.0}.get(unit, 1)
        vals[name] = v * scale
        kname = row.get("Kernel Name", kname)
    if "dram__bytes_read.sum" not in vals:
        return None, "ncu gave no dram metrics"
    t = vals["dram__bytes_read.sum"] + vals.get("dram__bytes_write.sum", 0.0)
    return {"traffic": t, "dram_read": vals["dram__bytes_read.sum"],
            "dram_write": vals.get("dram__bytes_write.sum"), "duration_s": vals.get("gpu__time_duration.sum"),
            "kernel": (kname or "").split("(")[0],
            "source": "measured in this run: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                      "--clock-control none (cache flushed) on launch 4 of a child process"}, None


def ncu_child(args):
    """--ncu-child: the same workload, 3 warm-up launches + 1 captured one."""
    import torch

    import paper_1103_4881_b200 as ds

    torch.cuda.set_device(0)
    cfg = workload(args, 1)
    d = make_downscaler(ds, args, cfg)
    x = ds.generate_frames(cfg["total"], d.in_frame_bytes, seed=args.seed)
    y = d.alloc_out(cfg["total"])
    for _ in range(4):
        d(x, y)
    torch.cuda.synchronize()
    return 0


def make_downscaler(ds, args, cfg):
    st = spec_stages(args)
    spec = None if st is None else ds.make_spec(h=st[0], v=st[1], chroma=cfg["chroma"])
    d = ds.Downscaler(cfg["w"], cfg["h"], cfg["channels"], chroma=cfg["chroma"], spec=spec)
    if args.kernel != "auto":
        d.set_kernel({"fused": ds.DS_KERNEL_FUSED, "fused_general": ds.DS_KERNEL_FUSED_GENERAL,
                      "generic": ds.DS_KERNEL_GENERIC}[args.kernel])
    if args.band_bytes:
        d.set_band_bytes(args.band_bytes)
    if args.stages or args.ctas:
        d.set_tuning(args.stages or 4, args.ctas)
    return d


def peer_probe():
    """--peer-probe (one process, GPUs 0 and 1): ds_run on GPU 0 storing into
    GPU 1's memory after ds_enable_peer must equal the local output.  bench.py
    runs this in a child before it enables the fused gather by default, so a
    peer-store fault cannot take the measured run down with it."""
    import torch

    import paper_1103_4881_b200 as ds

    if torch.cuda.device_count() < 2:
        print("probe: fewer than 2 GPUs")
        return 3
    torch.cuda.set_device(0)
    d = ds.Downscaler(1920, 1080, 3)
    x = ds.generate_frames(16, d.in_frame_bytes, seed=7)
    ref = d(x)
    d.enable_peer(1)
    y1 = torch.zeros((16, d.out_frame_bytes), dtype=torch.uint8, device="cuda:1")
    d(x, y1)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    ok = torch.equal(ref.cpu(), y1.cpu())
    print("probe:", "ok" if ok else "MISMATCH")
    return 0 if ok else 4


def cpu_oracle_sample(cfg, seed, budget_s, stages=None):
    """Time the CPU oracle (O1 tiler executor, plain C, 1 thread) on the first
    frames of the same stream until ~budget_s of work.  Test infrastructure:
    only this leg (and the verification leg) of bench.py touch oracle/."""
    import oracle
    import synth

    saved = os.sched_getaffinity(0)
    core = sorted(saved)[0]
    try:
        os.sched_setaffinity(0, {core})
    except Exception:
        core = None
    W, H, ch, chroma = cfg["w"], cfg["h"], cfg["channels"], cfg["chroma"]
    st = (None, None) if stages is None else tuple(oracle.stage_from_dict(s) for s in stages)
    times, k = [], 0
    t_all = time.perf_counter()
    try:
        while k < max(1, cfg["total"]) and (k < 2 or sum(times) < budget_s):
            fr = synth.random_frames(seed, k, 1, W, H, ch, chroma)
            t0 = time.perf_counter()
            oracle.execute_frames(fr, W, H, ch, chroma, *st)
            times.append(time.perf_counter() - t0)
            k += 1
        wall = time.perf_counter() - t_all
        per = statistics.median(times)
        o2 = None
        if stages is None:          # O2, the direct nested-loop oracle, default taps only
            o2_times = []
            for k2 in range(min(k, 5)):
                fr = synth.random_frames(seed, k2, 1, W, H, ch, chroma)
                t0 = time.perf_counter()
                oracle.direct_frames(fr, W, H, ch, chroma)
                o2_times.append(time.perf_counter() - t0)
            o2 = 1.0 / statistics.median(o2_times)
    finally:
        try:
            os.sched_setaffinity(0, saved)
        except Exception:
            pass
    return {
        "value": 1.0 / per, "unit": "frames/s", "cores": 1, "kind": "oracle",
        "sample": f"frames 0..{k - 1} of the same seeded stream ({k} frames), O1 tiler executor "
                  f"(oracle/ds_oracle.c, gcc -O2, 1 thread pinned to core {core}); "
                  f"median per-frame time {per * 1e3:.1f} ms; {wall:.1f} s of CPU work",
        "frames": k, "host_cpu": lscpu_model(), "o2_direct_value": o2, "oracle_core_id": core,
        "host_cores": os.cpu_count(),
    }


def lscpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, timed on the host cores;
    rank 0 only.  Each step = one frame of the workload through O1."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    import oracle
    import synth

    cfg = workload(args, world)
    W, H, ch, chroma = cfg["w"], cfg["h"], cfg["channels"], cfg["chroma"]
    stages = spec_stages(args)
    st = (None, None) if stages is None else tuple(oracle.stage_from_dict(s) for s in stages)
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
    except Exception:
        pass
    frames = [synth.random_frames(args.seed, k % cfg["total"], 1, W, H, ch, chroma)
              for k in range(min(args.steps + args.warmup, 8))]
    for k in range(args.warmup):
        oracle.execute_frames(frames[k % len(frames)], W, H, ch, chroma, *st)
    t0 = time.perf_counter()
    for k in range(args.steps):
        oracle.execute_frames(frames[k % len(frames)], W, H, ch, chroma, *st)
    dt = time.perf_counter() - t0
    fps = args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "u8",
        "data": f"synthetic (splitmix64 counter-hash frames by global byte index, seed {args.seed})",
        "config": config_dict(args, cfg, world),
        "step": "one frame of the workload through the CPU oracle (O1 tiler executor)",
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} frames (one per step) of the workload, O1 tiler "
                                   f"executor, plain C -O2, 1 thread, host {lscpu_model()}"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def time_steps(d, x, y, steps, graph, stream, clk):
    """The timed region: K ds_run calls (one CUDA graph replay, or per-call
    events), with >= CLOCK_WINDOW_MS of the same step replayed on each side
    for the clock sampler.  Returns (total_ms, per-launch ms list, host us)."""
    import torch

    def window(fn):
        t0 = time.perf_counter()
        while True:
            fn()
            torch.cuda.synchronize()
            if (time.perf_counter() - t0) * 1e3 >= CLOCK_WINDOW_MS:
                return

    host_call_us = None
    if graph:
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            d(x, y)                                   # warm the capture stream
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=cs):
            for _ in range(steps):
                d(x, y)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clk:
            window(g.replay)
            clk.mark("timed_start")
            e0.record(stream)
            g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            clk.mark("timed_end")
            window(g.replay)
        total_ms = e0.elapsed_time(e1)
        per = [total_ms / steps]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):                          # host cost of one un-captured call
            d(x, y)
        host_call_us = (time.perf_counter() - t0) / 200 * 1e6
        torch.cuda.synchronize()
        del g
    else:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * steps)]
        with clk:
            window(lambda: d(x, y))
            clk.mark("timed_start")
            for k in range(steps):
                evs[2 * k].record(stream)
                d(x, y)
                evs[2 * k + 1].record(stream)
            torch.cuda.synchronize()
            clk.mark("timed_end")
            window(lambda: d(x, y))
        per = [evs[2 * k].elapsed_time(evs[2 * k + 1]) for k in range(steps)]
        total_ms = evs[0].elapsed_time(evs[-1])
    return total_ms, per, host_call_us


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not (args.ncu_child or args.peer_probe):
        # `python bench.py --gpus N` outside torchrun: re-launch as N ranks on
        # this node (the same launch the driver uses), rendezvous on 127.0.0.1
        import socket

        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
               *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    if args.peer_probe:
        return peer_probe()
    if args.ncu_child:
        return ncu_child(args)
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1103_4881_b200 as ds
    from paper_1103_4881_b200.dist import gather_frames, padded_gather_rows, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # NCCL over NVLink for the real multi-GPU run; DS_DIST_BACKEND=gloo lets the
    # N>1 plumbing run with several ranks on one GPU (tests only: the ranks'
    # kernels never wait on one another, collectives go through the host).
    backend = os.environ.get("DS_DIST_BACKEND", "nccl")
    coll_dev = "cuda" if backend == "nccl" else "cpu"
    shared_gpu = False
    if world > 1:
        ndev = torch.cuda.device_count()
        shared_gpu = ndev < world
        torch.cuda.set_device(local % ndev)
        # the fused-gather probe (one process, GPUs 0/1) runs before any rank
        # touches the GPU heavily; rank 0 decides and broadcasts
        want_fused = args.fused_gather
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local % ndev))
        else:
            dist.init_process_group(backend)
        probe = torch.zeros(1, dtype=torch.int32, device=coll_dev)
        if rank == 0 and not args.no_gather and want_fused is not False:
            if shared_gpu or want_fused:
                probe[0] = 1                # ranks share one device: no peer stores involved
            else:
                try:
                    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--peer-probe"],
                                       capture_output=True, text=True, timeout=300, cwd=ROOT)
                    probe[0] = 1 if r.returncode == 0 else 0
                except Exception:
                    probe[0] = 0
        dist.broadcast(probe, 0)
        fused_gather_on = bool(int(probe[0]))
    else:
        torch.cuda.set_device(0)
        fused_gather_on = False
    dev = torch.cuda.current_device()

    cfg = workload(args, world)
    stages = spec_stages(args)
    fin, fout, fin_req = geometry(cfg, stages)
    lo, hi = shard_range(cfg["total"], world, rank)
    n = hi - lo
    m_rows = padded_gather_rows(cfg["total"], world) // world if world > 1 else n

    d = make_downscaler(ds, args, cfg)
    assert d.in_frame_bytes == fin and d.out_frame_bytes == fout
    stream = torch.cuda.current_stream()
    x = ds.generate_frames(n, fin, seed=args.seed, first_frame=lo)   # resident in HBM
    ybuf = torch.empty((max(m_rows, n), fout), dtype=torch.uint8, device=dev)   # padded for the gather
    y = ybuf[:n]
    torch.cuda.synchronize()

    # ---- warm-up (untimed) -------------------------------------------------
    for _ in range(max(args.warmup, 3)):
        d(x, y)
    torch.cuda.synchronize()
    kernel_used = d.last_kernel()

    # ---- timed region: K steps, CUDA events on the launching stream ---------
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(dev)
    total_ms, per, host_call_us = time_steps(d, x, y, args.steps, args.graph, stream, clk)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t = torch.tensor([total_ms, statistics.mean(per)], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, kern_ms = float(t[0]), float(t[1])

    frames_step = cfg["total"]
    frames_all = frames_step * args.steps
    fps = frames_all / (total_ms / 1e3)
    peak, peak_src = peaks()
    req_bytes = n * (fin_req + fout)             # required bytes per launch (per rank)
    achieved = req_bytes / (kern_ms / 1e3) / 1e9
    eff_full = n * (fin + fout) / (kern_ms / 1e3) / 1e9
    try:
        launch = d.launch_info(n, kernel_used)
    except Exception:
        launch = None

    # ---- N > 1: 1-GPU solo run of the same per-GPU workload (rank 0) --------
    solo = None
    if world > 1 and not args.no_solo:
        dist.barrier()
        if rank == 0:
            n1 = workload(args, 1)["total"]           # what `--gpus 1` of this command runs
            x1 = x if n1 == n else ds.generate_frames(n1, fin, seed=args.seed, first_frame=0)
            y1 = y if n1 == n else d.alloc_out(n1)
            for _ in range(3):
                d(x1, y1)
            torch.cuda.synchronize()
            solo_ms, _, _ = time_steps(d, x1, y1, args.steps, args.graph, stream, ClockSampler(dev))
            fps1 = n1 * args.steps / (solo_ms / 1e3)
            solo = {"fps_1gpu": fps1, "frames_1gpu": n1, "ms_per_step_1gpu": solo_ms / args.steps,
                    "speedup_vs_1gpu": fps / fps1,
                    "note": "rank 0 alone, same command at --gpus 1 (same frames per step as N = 1 "
                            "would run), timed the same way while the other ranks wait"
                            + ("; ranks share one GPU here, so this is not a scaling number"
                               if shared_gpu else "")}
            if x1 is not x:
                del x1, y1
                torch.cuda.empty_cache()
        dist.barrier()

    # ---- N > 1: gather to rank 0 (C-1), warmed up, repeated, timed ---------
    gather = None
    gathered = None
    if world > 1 and not args.no_gather:
        out = (torch.empty((padded_gather_rows(cfg["total"], world), fout), dtype=torch.uint8,
                           device="cuda" if backend == "nccl" else "cpu") if rank == 0 else None)
        src = ybuf[:m_rows] if backend == "nccl" else ybuf[:m_rows].cpu()
        gathered = gather_frames(src, cfg["total"], out=out)           # warm-up (communicators)
        torch.cuda.synchronize()
        times = []
        for _ in range(max(1, args.gather_reps)):
            dist.barrier()
            torch.cuda.synchronize()
            if backend == "nccl":
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gathered = gather_frames(src, cfg["total"], out=out)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            else:
                t0 = time.perf_counter()
                gathered = gather_frames(src, cfg["total"], out=out)
                times.append((time.perf_counter() - t0) * 1e3)
        gt = torch.tensor([statistics.median(times), min(times)], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gms = float(gt[0])
        step_ms = total_ms / args.steps
        gather = {"gather_ms": gms, "gather_ms_min": float(gt[1]), "reps": len(times),
                  "bytes": cfg["total"] * fout,
                  "gbs_into_rank0": cfg["total"] * fout / (gms / 1e3) / 1e9,
                  "with_gather_fps": frames_step / ((step_ms + gms) / 1e3),
                  "timing": ("CUDA events around dist.gather (NCCL) on the current stream, median of "
                             "reps after one warm-up gather, max over ranks" if backend == "nccl" else
                             "host wall time around dist.gather over gloo (host tensors), median of reps "
                             "after one warm-up, max over ranks"),
                  "method": "dist.gather of equal padded shards (one collective every rank enters)"}
        if rank != 0:
            gathered = None

    # ---- N > 1: gather fused into the kernels' stores (peer memory) ---------
    fused = None
    if world > 1 and not args.no_gather and fused_gather_on:
        from paper_1103_4881_b200.dist import share_rank0_tensor

        full = (torch.empty((cfg["total"], fout), dtype=torch.uint8, device=dev) if rank == 0 else None)
        full = share_rank0_tensor(full)
        d.enable_peer(full.device.index)
        view = full[lo:hi]
        d(x, view)                                     # warm
        torch.cuda.synchronize()
        dist.barrier()
        ks = max(1, args.gather_reps)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(ks):
            d(x, view)
        f1.record(stream)
        torch.cuda.synchronize()
        ft = torch.tensor([f0.elapsed_time(f1) / ks], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(ft, op=dist.ReduceOp.MAX)
        dist.barrier()
        fms = float(ft[0])
        ok = None
        if rank == 0 and gathered is not None:
            ok = bool(torch.equal(full.cpu(), gathered.cpu() if gathered.is_cuda else gathered))
        fused = {"ms": fms, "fps": frames_step / (fms / 1e3), "matches_gather": ok,
                 "method": "every rank's ds_run stores its frames into rank 0's buffer (CUDA IPC "
                           "+ ds_enable_peer): the transfer overlaps the filtering unit by unit"}
        dist.barrier()
        del view, full

    # ---- e2e: host pinned frames -> ds_run_host -> host, copies timed -------
    e2e = None
    if not args.no_e2e:
        hin = torch.empty((n, fin), dtype=torch.uint8, pin_memory=True)
        hin.copy_(x)
        hout = torch.empty((n, fout), dtype=torch.uint8, pin_memory=True)
        d.run_host(hin, hout)
        torch.cuda.synchronize()
        ks = max(1, args.e2e_steps)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ks):
            d.run_host(hin, hout)
        e1.record(stream)
        torch.cuda.synchronize()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=coll_dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        h2d_pf = (d.schedule_plan(ds.DS_SCHED_STREAMED)["h2d_bytes"] if stages is None else fin)
        e2e = {"value": frames_step * ks / (float(et[0]) / 1e3), "unit": "frames/s",
               "h2d_bytes_per_step": n * h2d_pf, "d2h_bytes_per_step": n * fout,
               "steps": ks, "api": "Downscaler.run_host -> ds_run_host (pinned host buffers)",
               "matches_device_path": bool(torch.equal(hout, y.cpu()))}
        del hin, hout

    # ---- every-frame parity against the oracle (rank 0) ---------------------
    parity = None
    if rank == 0 and not args.no_verify:
        from oracle.verify import verify_stream

        if world == 1:
            host, first = y.cpu().numpy(), lo
        elif gathered is not None:
            host, first = (gathered.cpu() if gathered.is_cuda else gathered).numpy(), 0
        else:
            host, first = y.cpu().numpy(), lo
        parity = verify_stream(host, cfg["w"], cfg["h"], cfg["channels"], cfg["chroma"], args.seed,
                               first_frame=first, stages=stages)
        parity["stream"] = ("the gathered stream on rank 0 (all ranks' frames)" if world > 1 and
                            gathered is not None else "this rank's output of the timed launch")
        parity["launch"] = "the bench launch configuration (the timed ds_run's output)"
        del host
    gathered = None

    # ---- CPU oracle baseline (rank 0) ---------------------------------------
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_oracle_sample(cfg, args.seed, args.cpu_seconds, stages)

    # ---- roofline.traffic: in-run ncu (N = 1) or the stamped committed capture
    key = args.config + ("" if args.spec == "spec" else f"_{args.spec}")
    want_ncu = args.ncu if args.ncu is not None else (world == 1)
    traffic = None
    if rank == 0 and world == 1 and want_ncu:
        traffic, why = ncu_measure(args)
        if traffic is None:
            traffic = {"error": why}
    build = source_hash()
    committed = ncu_committed(key if args.kernel == "auto" else f"{key}_{args.kernel}", n)
    if traffic is None or "traffic" not in traffic:
        if committed is not None:
            traffic = dict(traffic or {}, **committed)
            traffic["stale"] = committed.get("build") != build

    if rank == 0:
        kname = {ds.DS_KERNEL_FUSED: "ds_fused_band_kernel",
                 ds.DS_KERNEL_FUSED_GENERAL: ("ds_spec_kernel" if d.last_variant() == 2 else
                                              "ds_fused_general_kernel")}.get(kernel_used, "ds_generic_kernel")
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": cfg["scaling"],
            "vs_baseline": None, "dtype": "u8",
            "data": f"synthetic (splitmix64 counter-hash frames by global byte index, seed {args.seed})",
            "config": config_dict(args, cfg, world),
            "launch": dict(launch or {}, kernel_name=ds.KERNEL_NAMES.get(kernel_used),
                           variant_name=ds.VARIANT_NAMES.get((launch or {}).get("variant")),
                           frames_per_rank=n, band_groups=list(d.plan.band_groups)[: cfg["channels"]],
                           units_per_frame=d.plan.units_per_frame),
            "stages": (launch or {}).get("stages"),
            "ctas_per_sm": (launch or {}).get("ctas_per_sm"),
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": (traffic or {}).get("traffic"),
                "kernel": kname,
                "algorithmic_bytes_per_launch": req_bytes,
                "bytes_rule": ("per frame (8/9)*in + out: input rows 9g+4 carry zero V weight (S:540) "
                               "and are not required; see DESIGN.md" if stages is None else
                               "per frame in + out: every input row and column lies in some live tap "
                               "of the halo spec"),
                "avg_launch_ms": kern_ms,
                "peak_source": peak_src,
                "traffic_detail": traffic,
                "build": build,
                "effective_gbs_full_in_out": eff_full,
                "pct_of_8tbps_nominal_full_in_out": eff_full / 8000.0,
                "pct_of_measured_copy_full_in_out": eff_full / peak,
            },
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "per_launch": {
                "median_ms": statistics.median(per), "min_ms": min(per),
                "fps_median": n * world / (statistics.median(per) / 1e3),
                "fps_best": n * world / (min(per) / 1e3),
                "note": "rank 0's CUDA-event time of each timed ds_run (x world for the fps)"
                        if world > 1 else "CUDA-event time of each timed ds_run",
            } if not args.graph else None,
            "gpu_launches": args.steps,
            "clocks": clk.result(),
            "gather": gather,
            "gather_ms": (gather or {}).get("gather_ms"),
            "gather_fused": fused,
            "speedup_vs_1gpu": (solo or {}).get("speedup_vs_1gpu"),
            "solo_1gpu": solo,
            "timing": ("one CUDA graph of the K ds_run calls, replayed between two events"
                       if args.graph else "CUDA events around each ds_run on the launching stream"),
            "host_call_us": host_call_us,
            "impl": "ours",
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
