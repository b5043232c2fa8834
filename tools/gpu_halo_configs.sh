# the halo spec (--spec halo) on every bench geometry: one bench line each
mkdir -p gpurun_out; : > gpurun_out/halo_configs.jsonl
for cfg in ${CFGS:-hd420 hd444 4k420 cif420 sd420 qcif420}; do
  fr=""; case $cfg in cif420|sd420|qcif420) fr="--frames 2000";; esac
  timeout 300 python bench.py --spec halo --config $cfg $fr --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-ncu 2>/dev/null | grep '^{' >> gpurun_out/halo_configs.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/halo_configs.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], d["config"].get("frames"), round(d["value"]), round(d["roofline"]["frac"], 3),
          d["roofline"].get("kernel"), d["parity"]["bit_exact"] if d.get("parity") else None)
PY
