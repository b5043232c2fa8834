# A/B of K-N1g builds (VARIANTS) on misaligned-pointer planes (tools/k1g_coop_probe.py), REPS reps
mkdir -p gpurun_out; : > gpurun_out/coop_ab.txt
for i in $(seq ${REPS:-2}); do for v in $VARIANTS; do
  cp paper_1103_4881_b200/libds_$v.so paper_1103_4881_b200/libds.so
  echo "$v $(timeout 300 python tools/k1g_coop_probe.py | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(" ".join(f"{k.replace(chr(32),chr(95))}={v[chr(109)+chr(115)]:.3f}" for k,v in j.items()))')" >> gpurun_out/coop_ab.txt
done; done
