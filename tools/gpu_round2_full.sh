# Round-2 evidence run: full GPU test suite, the default and halo bench lines,
# the ncu launch list of the default bench command, an ncu --set full capture of
# K-N1 (default) and K-N1s (halo) -- each ncu pass only after its command exited 0.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_full.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --spec halo --steps 20 --warmup 5 > gpurun_out/bench_halo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_halo.log
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-verify --no-ncu"
$CMD > gpurun_out/plain_k1.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 20 --warmup 5 --no-ncu > gpurun_out/ncu_launches.log 2>&1
$CMD > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_band -s 3 -c 1 -o gpurun_out/prof_k1_hd420 $CMD > gpurun_out/ncu_k1.log 2>&1
$CMD --spec halo > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:ds_spec -s 3 -c 1 -o gpurun_out/prof_k1s_halo $CMD --spec halo > gpurun_out/ncu_k1s.log 2>&1
echo done
