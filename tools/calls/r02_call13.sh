set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_ata.py -k "fused or auto_plan" 2>&1 | tail -3
for c in c4 c3; do
timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-e2e --fuse-leaf-sums --no-autotune > gpurun_out/r02g_fused_$c.json 2>&1
timeout 400 python bench.py --config $c --steps 3 --warmup 2 --no-cpu --no-e2e --no-autotune > gpurun_out/r02g_plain_$c.json 2>&1
for f in fused plain; do python -c "
import json; d=json.load(open('gpurun_out/r02g_${f}_$c.json')); r=d['roofline']; print('$c $f', round(d['value']), 'frac', round(r['frac'],4), round(r['share_of_step'],4), round(r['secondary']['share_of_step'],4))"; done
done
