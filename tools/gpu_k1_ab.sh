# A/B of two libds.so builds in the same call (libds_new.so vs libds_old.so), interleaved, repeated
mkdir -p gpurun_out; : > gpurun_out/k1ab.txt
B="python bench.py --no-cpu-baseline --no-e2e --steps 300"
for rep in 1 2 3; do for cfg in ${AB_CONFIGS:-hd420 hd444 4k420}; do for v in new old; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  echo "$v $cfg $AB_EXTRA $(timeout 120 $B --config $cfg $AB_EXTRA | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["achieved"]), round(j["roofline"]["frac"],3), j["clocks"]["sm_mhz"], j["clocks"]["reasons"])')" >> gpurun_out/k1ab.txt
done; done; done
cp paper_1103_4881_b200/libds_new.so paper_1103_4881_b200/libds.so
