# SD / QCIF 4:2:0 (chroma rows W % 16 == 8): K-N1 (auto) vs K-N1g vs K-N2, 2000 frames
mkdir -p gpurun_out; : > gpurun_out/sd_qcif.jsonl
for cfg in sd420 qcif420; do for k in auto fused_general generic; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --config $cfg --frames 2000 --steps 50 --kernel $k >> gpurun_out/sd_qcif.jsonl
done; done
