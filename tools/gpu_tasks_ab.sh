# same-call A/B of libds_old.so vs libds_new.so on the task executor (H, shifted-origin H, V ms)
for rep in 1 2; do for v in old new; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  echo "$v $(timeout 120 python tools/general_perf.py --tasks 2>&1 | tail -1 | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["h"]["ds_run_task_flat_ms"],4), round(j["h"]["ds_run_task_wrapping_origin_ms"],4), round(j["v"]["ds_run_task_flat_ms"],4))')"
done; done
cp paper_1103_4881_b200/libds_new.so paper_1103_4881_b200/libds.so
