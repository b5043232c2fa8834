mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-e2e --steps 300 --warmup 5"
: > gpurun_out/sweep.txt
row() { echo "$* $(timeout 120 $B $* | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["achieved"]), round(j["roofline"]["frac"],3), j["config"]["grid"], j["config"]["block"], j["config"]["smem_bytes"], j["clocks"]["sm_mhz"])')" >> gpurun_out/sweep.txt; }
for st in 2 3 4 6; do for c in 1 2; do DS_UNIT_TARGET=32768 row --config hd420 --stages $st --ctas $c; done; done
for st in 2 3 4; do for c in 1 2 3; do DS_UNIT_TARGET=32768 row --config hd444 --stages $st --ctas $c; done; done
row --config hd420 --stages 4 --ctas 2
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --stages 4 --ctas 2"
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused_band -s 3 -c 1 -o gpurun_out/prof_v2 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
