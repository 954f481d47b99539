set -x
for v in head cur head cur; do
  if [ $v = head ]; then export ATA_LIB_PATH=_ab/head.so; else unset ATA_LIB_PATH; fi
  timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/ab_c4_$v.json 2> gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_$v.json')); r=d['roofline']
print('c4 $v', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), d['clocks'])"
done
