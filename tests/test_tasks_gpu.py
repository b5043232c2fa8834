"""GPU parity of the paper's unfused structure (K-N3: one kernel per
repetitive task, the u8 intermediate array in HBM) and of the
host transfer schedules -- against the CPU oracle, byte for
byte."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
ds = pytest.importorskip("paper_1103_4881_b200")

pytestmark = pytest.mark.gpu


def _same(got, want, what):
    if not np.array_equal(got, want):
        idx = np.argwhere(got != want)
        raise AssertionError(f"{what}: {len(idx)} bytes differ, first {idx[:3].tolist()}")


@pytest.mark.parametrize("W,H,ch,chroma", [(352, 288, 3, 1), (1920, 1080, 3, 1), (1920, 1080, 3, 0),
                                           (48, 27, 1, 1), (40, 45, 1, 1), (176, 144, 3, 1)])
def test_htask_vtask_match_oracle_mid_and_out(W, H, ch, chroma):
    d = ds.Downscaler(W, H, ch, chroma=chroma)
    fr = synth.random_frames(W, 0, 3, W, H, ch, chroma)
    mids, outs = oracle.execute_frames_mid(fr, W, H, ch, chroma)
    assert d.mid_frame_bytes == mids.shape[1]
    x = torch.from_numpy(fr).cuda()
    mid = d.htask(x)
    out = d.vtask(mid)
    torch.cuda.synchronize()
    _same(mid.cpu().numpy(), mids, "mid")
    _same(out.cpu().numpy(), outs, "out")


def test_tasks_plane_subsets_and_unaligned_mid():
    W, H = 352, 288
    d = ds.Downscaler(W, H, 3)
    fr = synth.random_frames(2, 0, 4, W, H)
    mids, outs = oracle.execute_frames_mid(fr, W, H)
    x = torch.from_numpy(fr).cuda()
    buf = torch.zeros(4 * d.mid_frame_bytes + 32, dtype=torch.uint8, device="cuda")
    mid = buf[2: 2 + 4 * d.mid_frame_bytes].view(4, -1)        # 2-byte aligned only
    out = torch.zeros((4, d.out_frame_bytes), dtype=torch.uint8, device="cuda")
    for p in (2, 0, 1):                                         # one plane at a time
        d.htask(x, mid, planes=(p, 1))
        d.vtask(mid, out, planes=(p, 1))
    torch.cuda.synchronize()
    _same(mid.cpu().numpy(), mids, "mid subsets")
    _same(out.cpu().numpy(), outs, "out subsets")


def test_generic_tasks_halo_spec():
    h = dict(pattern=13, paving=8, origin=3,
             weights=[[1, 2, 3, 0, 0, 0, 0, 0, 0, 0, 0, 1, 1], [0, 0, 0, 2, 2, 2],
                      [0, 0, 0, 0, 0, 0, 4, 4, 1, 1]], divisor=8, bias=4)
    v = dict(pattern=14, paving=9, origin=-5,
             weights=[[2, 2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 4], [0, 0, 4, 4],
                      [0, 0, 0, 0, 0, 3, 3, 0, 0, 0, 0, 2], [0, 0, 0, 0, 0, 0, 0, 5, 3]],
             divisor=8, bias=4)
    spec = ds.make_spec(h=h, v=v)
    d = ds.Downscaler(64, 36, 3, spec=spec)
    fr = synth.random_frames(8, 0, 2, 64, 36)
    oh = oracle.make_stage(13, 8, 3, h["weights"], 8, 4)
    ov = oracle.make_stage(14, 9, -5, v["weights"], 8, 4)
    mids, outs = oracle.execute_frames_mid(fr, 64, 36, 3, 1, oh, ov)
    x = torch.from_numpy(fr).cuda()
    mid = d.htask(x)
    out = d.vtask(mid)
    torch.cuda.synchronize()
    _same(mid.cpu().numpy(), mids, "generic mid")
    _same(out.cpu().numpy(), outs, "generic out")
    _same(d(x).cpu().numpy(), outs, "fused path on the same spec")


@pytest.mark.parametrize("sched", [0, 1, 2, 3])
@pytest.mark.parametrize("pinned", [True, False])
def test_schedules_produce_the_oracle_output(sched, pinned):
    W, H, n = 352, 288, 6
    d = ds.Downscaler(W, H, 3)
    fr = synth.random_frames(13, 0, n, W, H)
    hin = torch.from_numpy(fr)
    if pinned:
        hin = hin.pin_memory()
    d.set_host_chunk(4)
    hout, st = d.run_schedule(hin, sched)
    _same(hout.numpy(), oracle.execute_frames(fr, W, H), ds.SCHED_NAMES[sched])
    plan = d.schedule_plan(sched)
    assert st["frames"] == n
    if sched != ds.DS_SCHED_STREAMED:
        for k in ("h2d_count", "d2h_count", "h2d_bytes", "d2h_bytes", "launches"):
            assert st[k] == n * plan[k], k
        assert st["h2d_ms"] > 0 and st["d2h_ms"] > 0 and st["kernel_ms"] > 0
        assert st["total_ms"] >= 0.9 * (st["h2d_ms"] + st["d2h_ms"] + st["kernel_ms"])
    else:
        # the dead input row 9g+4 (zero V weight) is not transferred
        assert st["h2d_bytes"] == n * d.in_frame_bytes // 9 * 8 and st["h2d_count"] == 2


def test_schedule_zero_frames_and_errors():
    d = ds.Downscaler(352, 288, 3)
    hin = torch.zeros((0, d.in_frame_bytes), dtype=torch.uint8)
    out, st = d.run_schedule(hin, ds.DS_SCHED_NAIVE)
    assert st["frames"] == 0 and out.shape[0] == 0
    with pytest.raises(ds.DSError):
        d.run_schedule(torch.zeros((1, d.in_frame_bytes), dtype=torch.uint8), 7)
