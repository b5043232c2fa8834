# K-N1 launch shape with the driver's bench command (20 steps, graph replay):
# the default (2 CTAs/SM on HD, rings sharing 120 KB) vs 1 CTA/SM x 4 stages, interleaved, REPS times
mkdir -p gpurun_out; : > gpurun_out/k1_cta_ab.txt
for i in $(seq ${REPS:-5}); do
  for v in default one; do
    if [ $v = one ]; then X="--ctas 1 --stages 4"; else X=""; fi
    python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-ncu --no-verify $X 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']
print('$v', round(j['value']), round(r['frac'],4), j['ctas_per_sm'], j['stages'], j['clocks']['sm_mhz'], j['clocks']['reasons'])" >> gpurun_out/k1_cta_ab.txt
  done
done
cat gpurun_out/k1_cta_ab.txt
