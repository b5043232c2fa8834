# K-N1 band size x ring depth x CTAs/SM on the short-row formats (SD, CIF, QCIF 4:2:0,
# 300 frames, graph replay): is one CTA per SM with a deep ring right for them?
mkdir -p gpurun_out; : > gpurun_out/k1_small.txt
for cfg in ${CFGS:-sd420 cif420 qcif420}; do
B="python bench.py --no-cpu-baseline --no-e2e --steps 300 --config $cfg"
echo "$cfg default $(timeout 120 $B | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["frac"],3), j["config"]["smem_bytes"], j["config"]["band_groups"])')" >> gpurun_out/k1_small.txt
for bb in ${BANDS:-8192 16384 30720}; do for st in 2 3 4; do for ct in 1 2 3; do
  echo "$cfg band=$bb stages=$st ctas=$ct $(timeout 120 $B --band-bytes $bb --stages $st --ctas $ct 2>/dev/null | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["frac"],3), j["config"]["smem_bytes"], j["config"]["band_groups"], j["config"].get("grid"))' 2>/dev/null)" >> gpurun_out/k1_small.txt
done; done; done; done
