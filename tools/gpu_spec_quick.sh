# K-N1s quick loop: parity tests + halo timing (+ optional ncu capture with NCU=1)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_spec_kernel_gpu.py -x -q > gpurun_out/pytest_spec.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_spec.log
for i in 1 2; do timeout 300 python tools/spec_time.py; done > gpurun_out/spec_time.txt 2>&1
if [ -n "$NCU" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ds_spec -s 3 -c 1 -o gpurun_out/prof_spec python tools/spec_time.py > gpurun_out/ncu_spec.log 2>&1
fi
tail -2 gpurun_out/pytest_spec.log; cat gpurun_out/spec_time.txt
