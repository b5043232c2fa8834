# interleaved A/B on the headline config: the default launch shape vs the previous
# one (1 CTA/SM, 4-stage ring: --stages 4 --ctas 1), REPS reps
mkdir -p gpurun_out; : > gpurun_out/k1_hd_ab.txt
for i in $(seq ${REPS:-5}); do for arm in default one_cta; do
  X=""; [ $arm = one_cta ] && X="--stages 4 --ctas 1"
  echo "$arm $(timeout 120 python bench.py --no-cpu-baseline --no-e2e $X | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["frac"],4), j["config"]["grid"], j["clocks"]["sm_mhz"])')" >> gpurun_out/k1_hd_ab.txt
done; done
