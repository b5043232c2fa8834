# Round evidence on the current build: GPU parity tests, the default bench line,
# every other bench config, the reference arm, one-frame latency, and the N>1
# path as 2 ranks on one GPU (gloo; plumbing check only).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" > gpurun_out/status.txt
timeout 300 python bench.py > gpurun_out/bench_final.jsonl 2> gpurun_out/bench_final.err; echo "bench=$?" >> gpurun_out/status.txt
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_reference.jsonl 2>&1; echo "ref=$?" >> gpurun_out/status.txt
: > gpurun_out/configs.jsonl
for cfg in hd444 4k420 4k444 cif420 sd420 qcif420; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline >> gpurun_out/configs.jsonl 2>> gpurun_out/configs.err
done
: > gpurun_out/latency.jsonl
for extra in "--no-graph" "--graph"; do timeout 120 python bench.py --frames 1 --steps 2000 --no-cpu-baseline --no-e2e $extra >> gpurun_out/latency.jsonl 2>&1; done
DS_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --frames 600 --gather > gpurun_out/bench_2rank_gloo.log 2>&1; echo "bench2=$?" >> gpurun_out/status.txt
echo done >> gpurun_out/status.txt
