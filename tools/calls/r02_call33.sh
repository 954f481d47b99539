set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
ATA_RIDE_DEBUG=1 timeout 240 python tools/ride_check.py 2>&1 | sort | uniq -c | sort -rn | head -20
for r in 0 1; do
  ATA_RIDE=$r timeout 400 python bench.py --config c4 --steps 3 --warmup 2 --no-e2e --no-cpu --dump-units gpurun_out/ride${r}_units_c4.json > gpurun_out/ride${r}_bench_c4.json 2> gpurun_out/ride${r}_bench_c4.err
  tail -3 gpurun_out/ride${r}_bench_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ride${r}_bench_c4.json')); r=d['roofline']
print('c4 ride=$r', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), r['secondary']['share_of_step'], r['secondary']['riding']['executor_rides_per_step'])"
done
for b in 40 6; do
  timeout 400 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu --ws-budget $b > gpurun_out/ride_c3_b$b.json 2> gpurun_out/ride_c3_b$b.err
  tail -3 gpurun_out/ride_c3_b$b.err
  python -c "
import json; d=json.load(open('gpurun_out/ride_c3_b$b.json')); r=d['roofline']
print('c3 budget=$b', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), r['secondary']['share_of_step'], r['secondary']['riding']['executor_rides_per_step'])"
done
