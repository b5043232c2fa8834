# A/B of K-N1g: libds_old.so vs libds_new.so, tools/general_perf.py each, same call
mkdir -p gpurun_out
for v in old new; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  timeout 300 python tools/general_perf.py --out gpurun_out/general_perf_$v.json > /dev/null 2> gpurun_out/general_perf_$v.err
done
cp paper_1103_4881_b200/libds_new.so paper_1103_4881_b200/libds.so
