set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for r in 0 1; do
  ATA_RIDE=$r timeout 500 python bench.py --config c4 --steps 2 --warmup 1 --no-e2e --no-cpu --gain 1.0 --dump-units gpurun_out/g10_ride${r}_units.json > gpurun_out/g10_ride${r}.json 2> gpurun_out/g10_ride${r}.err
  tail -2 gpurun_out/g10_ride${r}.err
  python -c "
import json; d=json.load(open('gpurun_out/g10_ride${r}.json')); r=d['roofline']
print('c4 gain1.0 ride=$r', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), r['secondary']['share_of_step'])"
done
