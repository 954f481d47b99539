# full-size parity log with the RED ride + spread hoist, c5 sustained leg, ride capacity sweeps
set -x
rm -f gpurun_out/r02m_parity_fullsize.jsonl
ATA_PARITY_LOG=gpurun_out/r02m_parity_fullsize.jsonl timeout 1500 python -m pytest tests/test_gpu_configs.py -q 2>&1 | tail -4
cat gpurun_out/r02m_parity_fullsize.jsonl
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02m_bench_c5.json 2> gpurun_out/r02m_bench_c5.err
tail -3 gpurun_out/r02m_bench_c5.err
python -c "
import json; d=json.load(open('gpurun_out/r02m_bench_c5.json')); r=d['roofline']
print('c5', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'sustained', r.get('sustained'))"
for v in "" "--ride-gbs 550" "--ride-gbs 600" "--ride-gbs 700" "--ride-band-gb 0.6" "--ride-lookback 16" ""; do
  timeout 500 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c4_g.json 2> gpurun_out/ab_c4.err
  tail -2 gpurun_out/ab_c4.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c4_g.json')); r=d['roofline']
print('c4 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'])"
done
for v in "" "--ride-gbs 800" "--ride-gbs 500" ""; do
  timeout 500 python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu $v > gpurun_out/ab_c3_g.json 2> gpurun_out/ab_c3.err
  tail -2 gpurun_out/ab_c3.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c3_g.json')); r=d['roofline']
print('c3 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), r['secondary']['share_of_step'], d['config'].get('tuned'))"
done
