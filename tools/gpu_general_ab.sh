# A/B of K-N1g: libds_old.so vs libds_new.so, tools/general_perf.py each, same call,
# REPS repetitions; one line per run with every kernel's ms (gpurun_out/general_ab.txt)
mkdir -p gpurun_out; : > gpurun_out/general_ab.txt
for i in $(seq ${REPS:-2}); do for v in old new; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  timeout 300 python tools/general_perf.py --out gpurun_out/general_perf_$v.json > /dev/null 2> gpurun_out/general_perf_$v.err
  python - "$v" >> gpurun_out/general_ab.txt <<'PY'
import json, sys
v = sys.argv[1]
j = json.load(open(f"gpurun_out/general_perf_{v}.json"))
out = []
for cfg, d in j.items():
    if isinstance(d, dict):
        for k, x in d.items():
            if isinstance(x, dict) and "ms" in x and "K-N1g" in k:
                out.append(f"{cfg}={x['ms']:.4f}")
print(v, " ".join(out))
PY
done; done
cp paper_1103_4881_b200/libds_new.so paper_1103_4881_b200/libds.so
