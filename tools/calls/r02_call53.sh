# ride variants: cache policy of the store / reduction, pipelined rows, hybrid masks
set -x
for lib in cs pol polpipe cspipe cs7 cs_nored pipe mask7 pipe7; do
  ATA_LIB_PATH=_ab/$lib.so timeout 300 python tools/ride_ab.py bound 2>&1 | grep prods
done
HOIST="--ride-lookback 64 --ride-band-gb 1.25 --ride-arenas 1 --ride-gbs 650"
for lib in cs pol polpipe cspipe pipe; do
  ATA_LIB_PATH=_ab/$lib.so timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $HOIST > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$lib]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'])"
done
for lib in cs pol; do
  ATA_LIB_PATH=_ab/$lib.so timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu --ride-lookback 64 --ride-band-gb 1.25 --ride-arenas 1 --ride-gbs 1200 --gain 1.0 > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 gain1.0 [$lib]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'])"
done
