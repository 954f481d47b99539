set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 240 python tools/ride_check.py 2>&1 | tail -4
[ "${PIPESTATUS[0]}" = 0 ] || { echo "ride_check failed"; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_ride.py 2>&1 | tail -3
for v in "" "--gain 1.0"; do
  timeout 500 python bench.py --config c4 --steps 3 --warmup 2 --no-e2e --no-cpu $v --dump-units "gpurun_out/bulk_units_${v// /_}.json" > gpurun_out/bulk_c4.json 2> gpurun_out/bulk_c4.err
  tail -2 gpurun_out/bulk_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/bulk_c4.json')); r=d['roofline']
print('c4 bulk $v', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), r['secondary']['share_of_step'], d['plan']['mults_over_classical'])"
done
