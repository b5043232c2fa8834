set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default.log
timeout 600 python bench.py --spec halo --steps 20 --warmup 5 > gpurun_out/bench_halo.log 2>&1; echo "rc=$?" >> gpurun_out/bench_halo.log
DS_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_gloo2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_gloo2.log
tail -3 gpurun_out/*.log
