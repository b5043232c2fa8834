# K-N1 band size x ring depth sweep on hd420 (profiles/r01/k1_band_stage_sweep.txt)
mkdir -p gpurun_out; : > gpurun_out/k1s.txt
B="python bench.py --no-cpu-baseline --no-e2e --steps 300 --config hd420"
for bb in 16384 24576 32768 49152; do for st in 3 4 5 6 8; do
  echo "band=$bb stages=$st $(timeout 120 $B --band-bytes $bb --stages $st --ctas 1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["frac"],3), j["config"]["smem_bytes"], j["config"]["band_groups"], j["clocks"]["sm_mhz"])')" >> gpurun_out/k1s.txt
done; done
