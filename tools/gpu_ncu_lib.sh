# ncu --set full (source) of the K-N1g-family kernel in tools/spec_time.py with library variant $V
mkdir -p gpurun_out
cp paper_1103_4881_b200/libds_$V.so paper_1103_4881_b200/libds.so
python tools/spec_time.py > gpurun_out/plain_$V.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-ds_spec} -s 3 -c 1 -o gpurun_out/prof_$V python tools/spec_time.py > gpurun_out/ncu_$V.log 2>&1
echo "rc=$?"
