# private-partial tail split of large leaf groups: tests, same-box A/B on c4 / c3, intermediate gain
set -x
timeout 900 python -m pytest tests/test_gpu_ride.py tests/test_gpu_ata.py -q 2>&1 | tail -3
for v in "--no-tail-private" "" "--no-tail-private" "" "--gain 1.1" "--ride-gbs 2000"; do
  timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],4), 'adds', round(r['secondary']['share_of_step'],4), 'exec', r['executed_flops_per_step']/r['algorithmic_flops_per_step'])"
done
for v in "--no-tail-private" "" "--no-tail-private" ""; do
  timeout 500 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c3_g.json 2> gpurun_out/ab_c3.err
  tail -2 gpurun_out/ab_c3.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c3_g.json')); r=d['roofline']
print('c3 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],4), 'adds', round(r['secondary']['share_of_step'],4), d['config'].get('autotuned'))"
done
rm -f gpurun_out/r02n_parity_c4.jsonl
ATA_PARITY_LOG=gpurun_out/r02n_parity_c4.jsonl timeout 1200 python -m pytest tests/test_gpu_configs.py -q -k "c4 or c3" 2>&1 | tail -3
cat gpurun_out/r02n_parity_c4.jsonl
