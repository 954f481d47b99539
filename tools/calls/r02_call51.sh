# RIDE_RED A/B: riding sums as store + L2 reduction (no FP64-pipe adds) vs DADD
set -x
ATA_LIB_PATH=_ab/red.so timeout 600 python -m pytest tests/test_gpu_ride.py -q 2>&1 | tail -3
for lib in "" _ab/red.so; do
  ATA_LIB_PATH=$lib timeout 300 python tools/ride_ab.py 2>&1 | grep prods
done
for v in "" "--ride-gbs 1e9" "--gain 1.0 --ride-gbs 1e9" "--gain 1.0 --ride-gbs 2000"; do
 for lib in "" _ab/red.so; do
  ATA_LIB_PATH=$lib timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$lib] [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'])"
 done
done
