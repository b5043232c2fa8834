mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-e2e --steps 300 --warmup 5"
for st in 2 3 4 6; do for c in 1 2 3 0; do
  echo "stages=$st ctas=$c $(timeout 120 $B --stages $st --ctas $c | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["achieved"]), j["config"]["grid"], j["config"]["smem_bytes"], j["clocks"]["sm_mhz"])')" >> gpurun_out/sweep.txt
done; done
for cfg in hd444 4k420 4k444 cif420; do timeout 200 $B --config $cfg >> gpurun_out/configs.jsonl 2>&1; done
CMD="python bench.py --steps 10 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
CMD2="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD2 > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused_band -s 3 -c 1 -o gpurun_out/prof_fused $CMD2 > gpurun_out/ncu_full.log 2>&1
echo done
