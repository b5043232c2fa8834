# ncu evidence for the current build: launch list of the default bench command and a
# --set full capture of the fused kernel (each only after the same command exited 0)
mkdir -p gpurun_out
CMD="python bench.py"
$CMD > gpurun_out/plain_default.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
CMD2="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for cfg in ${NCU_CONFIGS:-hd420}; do
  $CMD2 --config $cfg > gpurun_out/plain_$cfg.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fused_band -s 3 -c 1 -o gpurun_out/prof_$cfg $CMD2 --config $cfg > gpurun_out/ncu_full_$cfg.log 2>&1
done
echo done
