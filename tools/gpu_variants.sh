# same-call A/B of libds_<v>.so variants (VARIANTS="a b c"), K-N1g quick timing, 3 rounds
mkdir -p gpurun_out; : > gpurun_out/variants.txt
for rep in 1 2 3; do for v in $VARIANTS; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  echo "$v $(timeout 120 python tools/general_perf.py --quick 2>&1 | tail -1)" >> gpurun_out/variants.txt
done; done
