set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
ATA_RIDE_DEBUG=1 timeout 240 python tools/ride_check.py 2>&1 | sort | uniq -c | sort -rn | head -20
timeout 900 python -m pytest -x -q tests/test_gpu_ride.py 2>&1 | tail -5
for b in 20 10; do
  timeout 400 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu --ws-budget $b > gpurun_out/ride_c3_b$b.json 2> gpurun_out/ride_c3_b$b.err
  tail -3 gpurun_out/ride_c3_b$b.err
  python -c "
import json; d=json.load(open('gpurun_out/ride_c3_b$b.json')); r=d['roofline']
print('c3 budget=$b', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), r['secondary']['share_of_step'], r['secondary']['riding']['executor_rides_per_step'])"
done
for v in "--max-depth 5 --gain 1.0" "--max-depth 5 --gain 0.8" "--gain 1.0"; do
  timeout 400 python bench.py --config c4 --steps 3 --warmup 2 --no-e2e --no-cpu $v > gpurun_out/ride_c4_v.json 2> gpurun_out/ride_c4_v.err
  tail -3 gpurun_out/ride_c4_v.err
  python -c "
import json; d=json.load(open('gpurun_out/ride_c4_v.json')); r=d['roofline']
print('c4 $v', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), r['secondary']['share_of_step'], r['secondary']['riding']['executor_rides_per_step'], d.get('plan'))"
done
