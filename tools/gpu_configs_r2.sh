# Every bench geometry on the current build (SPEC taps): the 4K lines at 1000 frames per GPU
# (configs[4]), the small frames at 2000, configs[3] (3000 HD frames), one-frame latency, and the
# reference arm (one line each, appended to gpurun_out/configs_r2.jsonl)
mkdir -p gpurun_out; : > gpurun_out/configs_r2.jsonl
for spec in "hd444 0" "4k420 0" "4k444 0" "cif420 2000" "sd420 2000" "qcif420 2000" "hd420 3000"; do
  set -- $spec
  fr=""; [ "$2" != 0 ] && fr="--frames $2"
  timeout 300 python bench.py --config $1 $fr --steps 20 --warmup 5 --no-cpu-baseline --no-ncu 2>/dev/null | grep '^{' >> gpurun_out/configs_r2.jsonl
done
for extra in "--no-graph" "--graph"; do timeout 120 python bench.py --frames 1 --steps 2000 --no-cpu-baseline --no-e2e --no-ncu --no-verify $extra 2>/dev/null | grep '^{' >> gpurun_out/configs_r2.jsonl; done
timeout 300 python bench.py --impl reference --steps 10 --warmup 2 2>/dev/null | grep '^{' >> gpurun_out/configs_r2.jsonl
python - <<'PY'
import json
for l in open("gpurun_out/configs_r2.jsonl"):
    d = json.loads(l)
    r = d.get("roofline") or {}
    print(d.get("impl", "ours"), d["config"].get("workload"), d["config"].get("frames"), round(d["value"]), d["unit"],
          r.get("frac"), d.get("ctas_per_sm"), d.get("stages"), (d.get("parity") or {}).get("bit_exact"),
          d.get("ms_per_step"), (d.get("clocks") or {}).get("reasons"))
PY
