set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -x -q tests/test_gpu_ata.py -k "fused or depth_first or auto_plan" 2>&1 | tail -5
timeout 120 python tools/f64_ab.py 58 4096 5 2>&1 | tail -3
for v in "" "--fuse-leaf-sums"; do
  timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e $v > gpurun_out/r02_c4_$v.json 2>&1; python -c "
import json,sys; d=json.load(open('gpurun_out/r02_c4_$v.json')); r=d['roofline']
print('c4 $v', round(d['value']), round(d['ms_per_step'],1), r['frac'], r['share_of_step'], r['secondary']['share_of_step'])"
  timeout 400 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e $v > gpurun_out/r02_c3_$v.json 2>&1; python -c "
import json,sys; d=json.load(open('gpurun_out/r02_c3_$v.json')); r=d['roofline']
print('c3 $v', round(d['value']), round(d['ms_per_step'],1), r['frac'], r['share_of_step'], r['secondary']['share_of_step'])"
done
