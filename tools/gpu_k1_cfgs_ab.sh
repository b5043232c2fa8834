# same-call A/B of K-N1 builds (VARIANTS) over configs (AB_CONFIGS), bench value / frac
mkdir -p gpurun_out; : > gpurun_out/k1cfg.txt
for rep in 1 2; do for cfg in ${AB_CONFIGS:-cif420 qcif420 sd420 hd420}; do for v in $VARIANTS; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  echo "$v $cfg $AB_EXTRA $(timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 100 --config $cfg $AB_EXTRA | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), round(j["roofline"]["frac"],3), j["config"]["block"])')" >> gpurun_out/k1cfg.txt
done; done; done
cp paper_1103_4881_b200/libds_new.so paper_1103_4881_b200/libds.so
