# bench lines (default, halo, QCIF/CIF x 2000) with wall time, and the run-time compilation probe
mkdir -p gpurun_out
for args in "" "--spec halo" "--config qcif420 --frames 2000" "--config cif420 --frames 2000"; do
  s=$(date +%s.%N)
  python bench.py --steps 20 --warmup 5 $args > gpurun_out/b.json 2> gpurun_out/b.err
  e=$(date +%s.%N)
  python -c "
import json,sys; j=json.loads(open('gpurun_out/b.json').read()); r=j['roofline']; t=r.get('traffic_detail') or {}
print('[$args] wall %.1fs' % ($e-$s), 'value', round(j['value']), 'frac', round(r['frac'],4), 'traffic', r['traffic'], t.get('kernel'), 'parity', j['parity']['bit_exact'], j['parity']['frames_checked'], 'clk', j['clocks']['sm_mhz'], j['clocks']['reasons'], j['clocks']['samples'])" >> gpurun_out/bench_check.txt
  cp gpurun_out/b.json "gpurun_out/bench_$(echo $args | tr ' -' '__').json"
done
python tools/jit_probe.py >> gpurun_out/bench_check.txt 2>&1
cat gpurun_out/bench_check.txt
