# c5: L2 access-policy window over the TF32 rounding rings (ATA_TF32_RING_PIN=1) vs default; DRAM traffic of both under ncu
set -x
for e in "" "ATA_TF32_RING_PIN=1" "" "ATA_TF32_RING_PIN=1"; do
  env $e timeout 400 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu --no-sustained > gpurun_out/ab_c5.json 2> gpurun_out/ab_c5.err
  tail -3 gpurun_out/ab_c5.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c5.json')); r=d['roofline']
print('c5 [$e]', round(d['value']), 'ms', round(d['ms_per_step'],3), 'frac', round(r['frac'],4), d['clocks'])"
done
timeout 300 python -m pytest tests/test_gpu_configs.py -q -k c5 2>&1 | tail -2
ATA_TF32_RING_PIN=1 timeout 300 python -m pytest tests/test_gpu_configs.py -q -k c5 2>&1 | tail -2
for e in "X=1" "ATA_TF32_RING_PIN=1"; do
  env $e timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:prod_tf32_2sm -c 3 --csv --log-file gpurun_out/r02o_c5_traffic_$e.csv python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu --no-sustained > /dev/null 2>&1
  grep -E "prod_tf32" gpurun_out/r02o_c5_traffic_$e.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | tail -8
done
