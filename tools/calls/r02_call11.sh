set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_kernels.py tests/test_gpu_ata.py -k "syrk or legacy or budget or golden or auto_plan" 2>&1 | tail -3
timeout 120 python tools/f64_ab.py 58 4096 5 2>&1 | tail -2
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r02e_bench_c4.json 2>&1
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/r02e_bench_c3.json 2>&1
for c in c4 c3; do python -c "
import json; d=json.load(open('gpurun_out/r02e_bench_$c.json')); r=d['roofline']; print('$c', round(d['value']), 'e2e', round(d['e2e']['value']), 'frac', round(r['frac'],4), r['share_of_step'])"; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02e_ref_arm.json 2> gpurun_out/r02e_ref_arm.err; tail -c 600 gpurun_out/r02e_ref_arm.json
