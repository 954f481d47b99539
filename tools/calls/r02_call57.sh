# default build = integer sign flip (no DADD in the ride): capacity probe, deeper Strassen trees on c4 / c3
set -x
timeout 600 python -m pytest tests/test_gpu_ride.py -q 2>&1 | tail -2
timeout 300 python tools/ride_ab.py bound2 2>&1 | grep "prods 58"
for v in "" "--gain 1.0 --ride-gbs 1200" "--gain 1.0 --ride-gbs 1e9" "--gain 0.8 --max-depth 5 --ride-gbs 1e9" "--gain 0.8 --max-depth 5 --ride-gbs 1500" "--gain 0.6 --max-depth 6 --min-dim 256 --ride-gbs 1e9" "--gain 1.0 --ride-gbs 1600"; do
  timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],4), 'adds', round(r['secondary']['share_of_step'],4), 'exec', r['executed_flops_per_step']/r['algorithmic_flops_per_step'])"
done
for v in "--no-autotune" "--no-autotune --gain 1.0 --ride-gbs 1e9" "--no-autotune --leaf-cols 2048 --ws-budget 7.4" "--no-autotune --leaf-cols 2048 --ws-budget 7.4 --gain 1.0 --ride-gbs 1e9" "--no-autotune --leaf-cols 2048 --ws-budget 7.4 --gain 0.8 --max-depth 5 --ride-gbs 1e9" "--no-autotune --leaf-cols 1024 --ws-budget 7.4 --gain 0.8 --max-depth 5 --ride-gbs 1e9"; do
  timeout 500 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c3_g.json 2> gpurun_out/ab_c3.err
  tail -2 gpurun_out/ab_c3.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c3_g.json')); r=d['roofline']
print('c3 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],4), 'adds', round(r['secondary']['share_of_step'],4), 'exec', r['executed_flops_per_step']/r['algorithmic_flops_per_step'])"
done
