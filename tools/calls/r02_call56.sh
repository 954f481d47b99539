# integer sign flip (no DADD left in the ride) + full-row fast path: A/B against the default build
set -x
ATA_LIB_PATH=_ab/flip.so timeout 600 python -m pytest tests/test_gpu_ride.py -q 2>&1 | tail -3
for lib in "" _ab/flip.so _ab/flippipe.so; do
  ATA_LIB_PATH=$lib timeout 300 python tools/ride_ab.py 2>&1 | grep "prods 58"
  ATA_LIB_PATH=$lib timeout 300 python tools/ride_ab.py bound 2>&1 | grep "prods 58"
done
for v in "" "--ride-gbs 800" "--ride-gbs 1000" "--gain 1.0 --ride-gbs 1200"; do
 for lib in "" _ab/flip.so _ab/flippipe.so; do
  ATA_LIB_PATH=$lib timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$lib] [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'])"
 done
done
