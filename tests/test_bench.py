"""bench.py's JSON contract: the reference arm (the CPU oracle, runs here)
and the workload / scaling labels on the CPU; the full line on the GPU."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _line(args, timeout=600):
    r = subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, timeout=timeout,
                       cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference: the oracle as it stands, one frame per step, on one
    core; the line carries the contract keys with e2e bytes zero."""
    j = _line(["--impl", "reference", "--config", "qcif420", "--steps", "3", "--warmup", "1"])
    assert j["impl"] == "reference" and j["unit"] == "frames/s" and j["value"] > 0
    assert j["higher_is_better"] is True and j["n_gpus"] == 1 and j["steps"] == 3
    cb = j["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == j["value"] and cb["sample"]
    assert j["e2e"] == {"value": j["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert "workload" in j["config"]


def test_workload_labels():
    """Weak scaling by default (300 HD frames per GPU; N = 1 is configs[2]),
    --frames fixes the total (strong at N > 1); 4K is configs[4] per GPU."""
    sys.path.insert(0, ROOT)
    import bench

    ns = lambda **kw: type("A", (), dict(dict(config="hd420", frames=0), **kw))()   # noqa: E731
    w1 = bench.workload(ns(), 1)
    assert w1["total"] == 300 and w1["scaling"] == "weak" and w1["name"].startswith("configs[2]")
    w8 = bench.workload(ns(), 8)
    assert w8["total"] == 2400 and w8["scaling"] == "weak"
    s8 = bench.workload(ns(frames=3000), 8)
    assert s8["total"] == 3000 and s8["scaling"] == "strong" and s8["name"].startswith("configs[3]")
    k1 = bench.workload(ns(config="4k420"), 1)
    assert k1["total"] == 1000 and k1["name"].startswith("configs[4]")
    one = bench.workload(ns(frames=1), 1)
    assert one["name"].startswith("configs[1]")


@pytest.mark.gpu
def test_bench_line_contract():
    """The default arm's line on a B200: every contract key, a roofline for
    the fused kernel, e2e through the host path, clocks sampled during the
    timed region, K launches."""
    j = _line(["--steps", "20", "--warmup", "3", "--cpu-seconds", "2"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "cpu_baseline",
              "gpu_launches", "clocks"):
        assert k in j, k
    assert j["steps"] == 20 and j["warmup"] >= 3 and j["gpu_launches"] == 20 and j["dtype"] == "u8"
    r = j["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = j["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["matches_device_path"] is True
    c = j["clocks"]
    assert c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    assert c["samples"] >= 20 and c["samples_in_timed_region"] >= 1
    cb = j["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] > 0
    p = j["parity"]
    assert p["frames_checked"] == p["frames_total"] == 300 and p["bit_exact"] is True
    assert j["stages"] >= 2 and j["ctas_per_sm"] >= 1
    # both arms print the same config object (the driver's same_config check)
    ref = _line(["--impl", "reference", "--steps", "2", "--warmup", "1"])
    assert ref["config"] == j["config"]


@pytest.mark.gpu
def test_bench_halo_spec_line():
    """--spec halo: the K-N1g kernel on the halo spec, roofline on in + out
    bytes, every frame checked against O1 with the spec's stages."""
    j = _line(["--spec", "halo", "--steps", "10", "--warmup", "3", "--cpu-seconds", "2", "--no-ncu"])
    assert j["roofline"]["kernel"] == "ds_spec_kernel" and j["launch"]["variant"] == 2
    fin, fout = j["config"]["in_frame_bytes"], j["config"]["out_frame_bytes"]
    assert j["roofline"]["algorithmic_bytes_per_launch"] == 300 * (fin + fout)
    p = j["parity"]
    assert p["bit_exact"] is True and p["frames_checked"] == 300 and p["oracle"].startswith("O1")
    ref = _line(["--impl", "reference", "--spec", "halo", "--steps", "2", "--warmup", "1"])
    assert ref["config"] == j["config"]


def test_config_dict_is_shared_by_both_arms():
    """Both arms build `config` with bench.config_dict from the same inputs."""
    sys.path.insert(0, ROOT)
    import bench

    for spec in ("spec", "halo"):
        a = bench.parse(["--spec", spec])
        cfg = bench.workload(a, 1)
        c = bench.config_dict(a, cfg, 1)
        assert c["in_frame_bytes"] == 3110400 and c["out_frame_bytes"] == 518400
    j = _line(["--impl", "reference", "--config", "qcif420", "--steps", "1", "--warmup", "0"])
    a = bench.parse(["--config", "qcif420"])
    assert j["config"] == bench.config_dict(a, bench.workload(a, 1), 1)


@pytest.mark.gpu
def test_bench_two_ranks_one_gpu_line():
    """The N > 1 bench path on one GPU (two torchrun ranks, gloo process group):
    max-over-ranks timing, the padded gather to rank 0 (warmed up, repeated),
    the fused gather (same device, no probe), the 1-GPU solo run, every
    gathered frame checked against the oracle, cpu_baseline on rank 0."""
    env = dict(os.environ, DS_DIST_BACKEND="gloo")
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--cpu-seconds", "1", "--no-ncu"], capture_output=True, text=True, timeout=900,
                       cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["scaling"] == "weak" and j["config"]["frames"] == 600
    g = j["gather"]
    assert g["reps"] == 5 and g["gather_ms"] > 0 and g["bytes"] == 600 * j["config"]["out_frame_bytes"]
    assert j["gather_fused"] is not None and j["gather_fused"]["matches_gather"] is True
    assert j["solo_1gpu"]["frames_1gpu"] == 300 and j["speedup_vs_1gpu"] > 0
    p = j["parity"]
    assert p["frames_checked"] == p["frames_total"] == 600 and p["bit_exact"] is True
    assert j["cpu_baseline"]["cores"] == 1
