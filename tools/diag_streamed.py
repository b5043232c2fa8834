import time, torch, json, sys
sys.path.insert(0, "/root/repo")
import paper_1103_4881_b200 as ds
torch.cuda.set_device(0)
W, H, n = 1920, 1080, 300
d = ds.Downscaler(W, H, 3)
x = ds.generate_frames(n, d.in_frame_bytes, seed=1)
hin = torch.empty((n, d.in_frame_bytes), dtype=torch.uint8, pin_memory=True); hin.copy_(x)
hout = torch.empty((n, d.out_frame_bytes), dtype=torch.uint8, pin_memory=True)
out = {}
def ev_time(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); a.record(); fn(); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b), (time.perf_counter() - t0) * 1e3
d.run_schedule(hin[:8], ds.DS_SCHED_STREAMED, hout[:8])
for i in range(3):
    _, st = d.run_schedule(hin, ds.DS_SCHED_STREAMED, hout)
    out[f"sched_streamed_{i}"] = st["total_ms"]
for i in range(3):
    out[f"run_host_{i}"] = ev_time(lambda: d.run_host(hin, hout))
for i in range(2):
    _, st = d.run_schedule(hin, ds.DS_SCHED_STREAMED, hout)
    out[f"sched_streamed_after_{i}"] = st["total_ms"]
print(json.dumps(out))
