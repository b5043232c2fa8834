# same-call A/B of libds_<v>.so variants (VARIANTS="a b c") on the general task executor
mkdir -p gpurun_out; : > gpurun_out/variants_tasks.txt
for rep in 1 2; do for v in $VARIANTS; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  echo "$v $(timeout 120 python tools/general_perf.py --tasks 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["h"]["ds_run_task_flat_ms"],4), round(j["v"]["ds_run_task_flat_ms"],4))')" >> gpurun_out/variants_tasks.txt
done; done
