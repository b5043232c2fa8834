# K-N1 launch shape vs launch length: HD 3000 frames, 4K 300 frames (driver-style bench, graph replay)
mkdir -p gpurun_out; : > gpurun_out/k1_cta_ab3.txt
for spec in ${SPECS:-"hd420 3000" "4k420 300" "4k444 300" "hd420 1200"}; do
set -- $spec
for i in 1 2; do
  for v in default one; do
    if [ $v = one ]; then X="--ctas 1 --stages 4"; else X=""; fi
    python bench.py --config $1 --frames $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-ncu --no-verify $X 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']
print('$1 $2', '$v', round(j['value']), round(r['frac'],4), j['ctas_per_sm'], j['stages'], j['clocks']['sm_mhz'], j['clocks']['reasons'])" >> gpurun_out/k1_cta_ab3.txt
  done
done
done
cat gpurun_out/k1_cta_ab3.txt
