# round-2 validation: smoke, the whole -m gpu suite, every config's bench line
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 3000 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r02_final_gpu_tests.log
cat gpurun_out/r02_final_gpu_tests.log
for c in c1 c2 c3 c5 c4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r02_final_bench_$c.json 2> gpurun_out/r02_final_bench_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/r02_final_bench_$c.json')); r=d['roofline']
print('$c', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), 'e2e', round(d['e2e']['value']), 'cpu', round(d['cpu_baseline']['value'],1), d['clocks'])"
done
