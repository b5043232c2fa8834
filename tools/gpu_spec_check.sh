# K-N1s: parity tests (spec kernel + the K-N1g fuzz), halo timing, the SD halo
# bench line, and an ncu --set full capture of the halo kernel with NCU=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_spec_kernel_gpu.py tests/test_parity_gpu.py -x -q -k "spec or general or fuzz" > gpurun_out/pytest_spec.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_spec.log
for i in 1 2; do timeout 300 python tools/spec_time.py >> gpurun_out/spec_time.log 2>&1; done
timeout 300 python bench.py --spec halo --steps 20 --warmup 5 > gpurun_out/bench_halo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_halo.log
timeout 300 python bench.py --spec halo --config sd420 --frames 2000 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_halo_sd.log 2>&1; echo "rc=$?" >> gpurun_out/bench_halo_sd.log
if [ "$NCU" = 1 ]; then
CMD="python bench.py --spec halo --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-verify --no-ncu"
$CMD > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:ds_spec -s 3 -c 1 -o gpurun_out/prof_k1s_halo $CMD > gpurun_out/ncu_k1s.log 2>&1
fi
tail -3 gpurun_out/pytest_spec.log; cat gpurun_out/spec_time.log
