# ncu --set full captures of the non-headline kernels (K-N3 tasks, K-N1g, ds_task_kernel)
# via tools/prof_cases.py, each only after the same command exited 0 without ncu
mkdir -p gpurun_out
for w in tasks general runtask; do
  python tools/prof_cases.py $w > gpurun_out/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"htask|vtask|general|task_kernel" -s 2 -c 2 -o gpurun_out/prof_$w python tools/prof_cases.py $w > gpurun_out/ncu_$w.log 2>&1
done
echo done
