# RED ride as default: tests, multi-group hoist / bands / arenas A/B on c4, ride ingredient probes
set -x
timeout 900 python -m pytest tests/test_gpu_ride.py tests/test_gpu_ata.py -q 2>&1 | tail -3
for v in "" "--ride-lookback 64 --ride-band-gb 1.25" "--ride-lookback 64 --ride-band-gb 1.25 --ride-arenas 1" "--ride-lookback 64 --ride-band-gb 1.25 --ride-arenas 1 --ride-gbs 1000" "--ride-lookback 64 --ride-band-gb 1.25 --ride-arenas 1 --ride-gbs 650" ""; do
  timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'])"
done
for lib in "" _ab/noload.so _ab/nostore.so _ab/nored.so _ab/dadd.so; do
  ATA_LIB_PATH=$lib timeout 300 python tools/ride_ab.py bound 2>&1 | grep prods
done
