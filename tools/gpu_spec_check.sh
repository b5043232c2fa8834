# K-N1s: parity tests, the halo bench line, and an ncu --set full capture (after the bench exits 0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_spec_kernel_gpu.py -x -q > gpurun_out/pytest_spec.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_spec.log
timeout 300 python bench.py --spec halo --steps 20 --warmup 5 --no-ncu --cpu-seconds 2 > gpurun_out/bench_halo_spec.log 2>&1; echo "rc=$?" >> gpurun_out/bench_halo_spec.log
CMD="python bench.py --spec halo --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-verify --no-ncu"
$CMD > gpurun_out/plain_spec.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:ds_spec -s 3 -c 1 -o gpurun_out/prof_spec_halo $CMD > gpurun_out/ncu_spec.log 2>&1
echo "ncu rc=$?"
