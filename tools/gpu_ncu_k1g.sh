# ncu --set full (source-level) of K-N1g on the halo spec, after the same command exits 0 without ncu
mkdir -p gpurun_out
CMD="python bench.py --spec halo --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-verify --no-ncu"
TAG=${TAG:-k1g_halo}
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused_general -s 3 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo "rc=$?"
