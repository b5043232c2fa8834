# same-call A/B of library builds libds_<v>.so for v in $VARIANTS, REPS times:
# one line per run from tools/spec_time.py (or $TOOL) -> gpurun_out/lib_ab.txt
mkdir -p gpurun_out; : > gpurun_out/lib_ab.txt
cp paper_1103_4881_b200/libds.so /tmp/libds_keep.so
for i in $(seq ${REPS:-2}); do for v in $VARIANTS; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  echo "$v $(timeout 300 python ${TOOL:-tools/spec_time.py} 2>&1 | tail -1)" >> gpurun_out/lib_ab.txt
done; done
cp /tmp/libds_keep.so paper_1103_4881_b200/libds.so
cat gpurun_out/lib_ab.txt
