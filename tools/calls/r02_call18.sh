set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_ata.py tests/test_gpu_acceptance.py tests/test_gpu_callers.py 2>&1 | tail -4
for c in c2 c1 c4; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/r02j_bench_$c.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r02j_bench_$c.json')); r=d['roofline']
print('$c', round(d['value']), 'ms', round(d['ms_per_step'],2), 'frac', round(r['frac'],4), 'share', round(r['share_of_step'],3), 'e2e', round(d['e2e']['value']))"
done
