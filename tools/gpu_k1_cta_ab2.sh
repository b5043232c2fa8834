# K-N1 launch shape A/B over configs with the driver's bench command (graph replay):
# default vs 1 CTA/SM x 4 stages, interleaved, REPS times per config
mkdir -p gpurun_out; : > gpurun_out/k1_cta_ab2.txt
for cfg in ${CFGS:-hd444 4k420 cif420 hd420}; do
for i in $(seq ${REPS:-3}); do
  for v in default one; do
    if [ $v = one ]; then X="--ctas 1 --stages 4"; else X=""; fi
    python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-ncu --no-verify $X 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']
print('$cfg', '$v', round(j['value']), round(r['frac'],4), j['ctas_per_sm'], j['stages'], j['clocks']['sm_mhz'], j['clocks']['reasons'])" >> gpurun_out/k1_cta_ab2.txt
  done
done
done
cat gpurun_out/k1_cta_ab2.txt
