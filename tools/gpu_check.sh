# parity tests + default bench line + per-config bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" > gpurun_out/status.txt
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?" >> gpurun_out/status.txt
: > gpurun_out/configs.jsonl
for cfg in hd444 4k420 4k444 cif420; do timeout 200 python bench.py --config $cfg --no-cpu-baseline --no-e2e >> gpurun_out/configs.jsonl 2>&1; done
echo done
