# last check of HEAD: smoke, whole -m gpu suite, default bench line + reference arm
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 3000 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/r02p_gpu_tests.log
cat gpurun_out/r02p_gpu_tests.log
timeout 900 python bench.py > gpurun_out/r02p_bench_default.json 2> gpurun_out/r02p_bench_default.err
tail -2 gpurun_out/r02p_bench_default.err
python -c "
import json; d=json.load(open('gpurun_out/r02p_bench_default.json')); r=d['roofline']
print('default', d['config'], round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), 'e2e', round(d['e2e']['value']), 'cpu', round(d['cpu_baseline']['value'],1), d['clocks'], d['gpu_launches'])"
