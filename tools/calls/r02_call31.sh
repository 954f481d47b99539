set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 200 python tools/ride_debug.py 2050 1100 0.005 0 2>&1 | tail -12
timeout 200 python tools/ride_debug.py 2050 1100 0.005 1 2>&1 | tail -12
ATA_RIDE=0 timeout 200 python tools/ride_debug.py 2050 1100 0.005 1 2>&1 | tail -12
for r in 0 1; do
  ATA_RIDE=$r timeout 400 python bench.py --config c4 --steps 3 --warmup 2 --no-e2e --no-cpu --dump-units gpurun_out/ride${r}_units_c4.json > gpurun_out/ride${r}_bench_c4.json 2> gpurun_out/ride${r}_bench_c4.err
  tail -3 gpurun_out/ride${r}_bench_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ride${r}_bench_c4.json')); r=d['roofline']
print('c4 ride=$r', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3))"
done
