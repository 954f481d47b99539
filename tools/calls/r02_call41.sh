set -x
timeout 240 python tools/ride_check.py 2>&1 | tail -2
timeout 900 python -m pytest -x -q tests/test_gpu_ride.py 2>&1 | tail -2
timeout 300 python tools/ride_ab.py bound 2>&1 | grep prods
timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/reg2_c4.json 2> gpurun_out/reg2_c4.err
python -c "
import json; d=json.load(open('gpurun_out/reg2_c4.json')); r=d['roofline']
print('c4', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), r['secondary']['share_of_step'])"
