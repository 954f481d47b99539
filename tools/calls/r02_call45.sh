set -x
for v in "--ride-gbs 900" "--ride-gbs 1e9" "--ride-gbs 1200" "--ride-gbs 900" "--ride-gbs 1e9"; do
  timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'])"
done
for v in "--ride-gbs 900" "--ride-gbs 1e9" "--ride-gbs 900 --no-diag-first" "--ride-gbs 900" "--ride-gbs 1e9"; do
  timeout 500 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu --no-autotune --leaf-cols 2048 --ws-budget 10.5 $v > gpurun_out/ab_c3_g.json 2> gpurun_out/ab_c3.err
  tail -2 gpurun_out/ab_c3.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c3_g.json')); r=d['roofline']
print('c3 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'])"
done
