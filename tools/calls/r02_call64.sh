# c3 e2e: autotuned plan parameters vs the defaults under the three-block host pipeline
set -x
for v in "" "--no-autotune"; do
  timeout 600 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu $v > gpurun_out/ab_c3_e2e.json 2> gpurun_out/ab_c3_e2e.err
  tail -2 gpurun_out/ab_c3_e2e.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_c3_e2e.json'))
print('c3 [$v]', round(d['value']), 'ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value']), round(d['e2e']['ms_per_step'],1), d['config'].get('autotuned'))"
done
