set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for lib in "" _ab/fbk24.so _ab/fbk8.so; do
  ATA_LIB_PATH=$lib timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --fuse-leaf-sums > gpurun_out/r02i.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/r02i.json')); r=d['roofline']; print('fused $lib', round(d['value']), 'frac', round(r['frac'],4), round(r['share_of_step'],4), round(r['secondary']['share_of_step'],4))"
done
