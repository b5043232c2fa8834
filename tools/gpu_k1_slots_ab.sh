# same-call A/B of K-N1 output-ring depth (libds_s2.so: 2 slots, lets HD fit 3 CTAs/SM;
# libds_s3.so: 3 slots) over configs, REPS reps; leaves libds_s3.so installed
mkdir -p gpurun_out; : > gpurun_out/k1_slots.txt
for rep in $(seq ${REPS:-3}); do for cfg in ${AB_CONFIGS:-hd420 hd444 4k420 sd420 cif420}; do for v in s2 s3; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  echo "$v $cfg $(timeout 120 python bench.py --no-cpu-baseline --no-e2e --config $cfg | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["frac"],4), j["config"]["grid"], j["config"]["smem_bytes"], j["clocks"]["sm_mhz"])')" >> gpurun_out/k1_slots.txt
done; done; done
cp paper_1103_4881_b200/libds_s3.so paper_1103_4881_b200/libds.so
