# A/B of two libds.so builds in the same call: $1 = alternate .so path (built from another revision)
mkdir -p gpurun_out; : > gpurun_out/k1ab.txt
B="python bench.py --no-cpu-baseline --no-e2e --steps 300"
for rep in 1 2 3; do for cfg in hd420 hd444 4k420; do for v in new old; do
  if [ $v = old ]; then cp paper_1103_4881_b200/libds_old.so paper_1103_4881_b200/libds.so; else cp paper_1103_4881_b200/libds_new.so paper_1103_4881_b200/libds.so; fi
  echo "$v $cfg $(timeout 120 $B --config $cfg | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["achieved"]), round(j["roofline"]["frac"],3), j["clocks"]["sm_mhz"], j["clocks"]["reasons"])')" >> gpurun_out/k1ab.txt
done; done; done
cp paper_1103_4881_b200/libds_new.so paper_1103_4881_b200/libds.so
