mkdir -p gpurun_out
: > gpurun_out/gen_sweep.txt
for cfg in "8 2 2" "16 2 1"; do set -- $cfg
  echo "ncw=$1 stages=$2 ctas=$3 $(DS_GEN_NCW=$1 DS_GEN_STAGES=$2 DS_GEN_CTAS=$3 timeout 200 python tools/general_perf.py --out gpurun_out/gp.json | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["hd420_300_halo_spec"]["K-N1g fused band, any spec (TMA ring, smem halo + mid)"]["ms"],3), round(j["hd420_300_spec_taps"]["K-N1g fused band, any spec (TMA ring, smem halo + mid)"]["ms"],3), round(j["hd420_300_spec_taps"]["K-N1 fused band (TMA ring)"]["ms"],4))')" >> gpurun_out/gen_sweep.txt
done
