# usage: bash tools/gpu_sweep.sh  -- parity tests, then a stages x CTAs/SM sweep + other configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" > gpurun_out/status.txt
B="python bench.py --no-cpu-baseline --no-e2e --steps 300 --warmup 5"
: > gpurun_out/sweep.txt
for cfg in ${CONFIGS:-hd420 4k420}; do for st in ${STAGES:-2 3 4}; do for c in ${CTAS:-2 3 4 0}; do
  echo "$cfg stages=$st ctas=$c $(timeout 120 $B --config $cfg --stages $st --ctas $c | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["achieved"]), round(j["roofline"]["frac"],3), j["config"]["grid"], j["config"]["block"], j["config"]["smem_bytes"], j["clocks"]["sm_mhz"])')" >> gpurun_out/sweep.txt
done; done; done
echo done
