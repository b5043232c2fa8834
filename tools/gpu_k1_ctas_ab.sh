# interleaved A/B: K-N1 default launch shape vs 2-deep ring at up to 3 CTAs/SM (REPS reps)
mkdir -p gpurun_out; : > gpurun_out/k1_ctas_ab.txt
for i in $(seq ${REPS:-3}); do for cfg in ${CFGS:-hd420 hd444}; do for arm in default multi; do
  X=""; [ $arm = multi ] && X="--stages 2 --ctas 3"
  echo "$cfg $arm $(timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 300 --config $cfg $X | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["frac"],4), j["config"]["grid"], j["clocks"]["sm_mhz"])')" >> gpurun_out/k1_ctas_ab.txt
done; done; done
